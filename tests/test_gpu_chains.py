"""GPU chain parity: each mmFHE chain through mmfhe_eval_chain must reproduce
the oracle circuit's output residues bit for bit with an identical op trace
(north_star gate 1; Theorem P:999-1006), on seeded radar-shaped inputs
encrypted by the oracle client.  Full-size configs: C1 (k1_energy, PS1) and
C3 (k3_doppler_dft, PS3)."""
import numpy as np
import pytest

from oracle import ckks as orc
from oracle import circuits as cc
from oracle import dsp
from synth import radar
from synth.params import ps1, ps3, toy

from gpu_util import ct_in, ct_out, make_ctx, residues

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m(cuda_ctx_ok):
    from paper_2603_22437_b200 import build, mmfhe
    build.build()
    return mmfhe


def _mcfg(m, cfg: cc.ChainCfg, bins=(), taps=()):
    return m.chain_cfg(R=cfg.R, D=cfg.D, A=cfg.A, F=cfg.F, gamma=cfg.gamma, p_phi=cfg.p_phi,
                       taylor_order=cfg.taylor_order, n_slots=cfg.n_slots, bsgs_baby=cfg.bsgs_baby,
                       fc_dims=cfg.fc_dims, notch_width=cfg.notch_width, bands_bins=bins,
                       n_taps=[len(t) for t in taps], fs=cfg.fs, frame_batch=cfg.frame_batch, hoist=cfg.hoist,
                       vp_plus=cfg.vp_plus, iq_pack=cfg.iq_pack, lanes=cfg.lanes, cplx=cfg.cplx,
                       bsgs_aligned=cfg.bsgs_aligned, rotsum_inner=cfg.rotsum_inner,
                       rotsum_hoist_all=cfg.rotsum_hoist_all, ks_merge=cfg.ks_merge,
                       k1_conj_fuse=cfg.k1_conj_fuse)


def _run(m, P, keys, book, chain, cfg, cts, want, scalars=None, bins=(), taps=()):
    ctx = make_ctx(m, P, keys, book, scalars)
    mcfg = _mcfg(m, cfg, bins, taps)
    levels = ctx.chain_plan(chain, mcfg, cts[0].level, len(cts))
    assert levels == [w.level for w in want]
    outs = [ct_out(m, P, lv) for lv in levels]
    n = ctx.eval_chain(chain, mcfg, [ct_in(m, P, c) for c in cts], outs)
    assert n == len(want)
    for o, w in zip(outs, want):
        assert np.array_equal(residues(o), np.stack(w.c)), "residues differ from the oracle"
        assert o.scale == w.scale and o.level == w.level
    return ctx


def _vital_inputs(P, keys, cfg, lvl, seed):
    z, _ = radar.vital_scene(cfg.R, cfg.F, cfg.fs, seed=seed)
    zt = radar.preprocess_vital(z)
    cts = []
    for t in range(cfg.F):
        for part in (zt[t].real, zt[t].imag):
            cts.append(orc.encrypt_vector(P, keys, radar.pack_vital(part, cfg.n_slots), lvl, seed=seed + 1,
                                          index=len(cts)))
    return zt, cts


def test_k1_energy_c1_full_size(m):
    """C1: K1 only, N=2^13, 3 RNS limbs (2 Q + 1 P), R=64, F=32, depth 1."""
    P = ps1()
    cfg = cc.ChainCfg(R=64, F=32, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=3001)
    zt, cts = _vital_inputs(P, keys, cfg, 1, 3002)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    E = cc.k1_energy(ev, cts[0::2], cts[1::2])
    ctx = _run(m, P, keys, None, "k1_energy", cfg, cts, [E])
    assert ctx.trace() == ev.trace
    E_dec = orc.decrypt_vector(P, keys, E)[: cfg.R]
    want = dsp.energy(zt)
    assert np.max(np.abs(E_dec - want)) <= 1e-3 * np.max(np.abs(want))


def test_k1_energy_multi_session(m):
    """C1/C5 serving shape: S sessions in one call, batched over sessions."""
    P = toy(log_n=11, n_q=3, scale_bits=40, n_p=1, alpha=1)
    cfg = cc.ChainCfg(R=16, F=4, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=3011)
    sessions, cts = [], []
    for s in range(3):
        _, c = _vital_inputs(P, keys, cfg, 1, 3020 + 10 * s)
        sessions.append((c[0::2], c[1::2]))
        cts += c
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    want = cc.k1_energy_sessions(ev, sessions)
    ctx = _run(m, P, keys, None, "k1_energy", cfg, cts, want)
    assert ctx.trace() == ev.trace


def test_k1_energy_multi_session_host_outputs(m):
    """Batched export (one INTT per output batch) into host and device output buffers, and
    NTT-form outputs: the same residues as the oracle (coefficient form) in every case."""
    P = toy(log_n=11, n_q=3, scale_bits=40, n_p=1, alpha=1)
    cfg = cc.ChainCfg(R=16, F=2, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=3041)
    sessions, cts = [], []
    for s in range(4):
        _, c = _vital_inputs(P, keys, cfg, 1, 3050 + 10 * s)
        sessions.append((c[0::2], c[1::2]))
        cts += c
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    want = cc.k1_energy_sessions(ev, sessions)
    ctx = make_ctx(m, P, keys)
    mcfg = _mcfg(m, cfg)
    levels = ctx.chain_plan("k1_energy", mcfg, 1, len(cts))
    ins = [ct_in(m, P, c) for c in cts]
    for device in (False, True):
        outs = [ct_out(m, P, lv, device=device) for lv in levels]
        assert ctx.eval_chain("k1_energy", mcfg, ins, outs) == len(want)
        for o, w in zip(outs, want):
            assert np.array_equal(residues(o), np.stack(w.c))
            assert o.scale == w.scale and o.level == w.level
    # NTT-form device outputs, converted back through the library's own INTT
    outs = [ct_out(m, P, lv) for lv in levels]
    for o in outs:
        o.form = m.FORM_EVAL
    ctx.eval_chain("k1_energy", mcfg, ins, outs)
    for o, w in zip(outs, want):
        ctx.ntt(o.data.view(-1, P.n), [i % (o.level + 1) for i in range(2 * (o.level + 1))], inverse=True)
        assert np.array_equal(residues(o), np.stack(w.c))


def test_k3_multi_frame_batches(m):
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    cfg = cc.ChainCfg(A=2, R=4, D=8, F=3, n_slots=64, frame_batch=2, hoist=1)
    keys = orc.keygen(P, seed=3031, rotations=cc.required_rotations("k3_doppler_dft", cfg, P.n))
    rng = np.random.default_rng(3)
    cts = [orc.encrypt_vector(P, keys, rng.uniform(-1, 1, 64), P.L, seed=3032, index=i) for i in range(6)]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    want = []
    for s, e in cc.chunks(3, 2):
        dre, dim = cc.k3_doppler_dft_frames(ev, book, cts[2 * s:2 * e:2], cts[2 * s + 1:2 * e:2], cfg)
        want += dre + dim
    ctx = _run(m, P, keys, book, "k3_doppler_dft", cfg, cts, want)
    assert ctx.trace() == ev.trace


def test_vitals_v1_small(m):
    P = toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)
    cfg = cc.ChainCfg(R=16, F=6, gamma=2, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=3101, rotations=cc.required_rotations("vitals_v1", cfg, P.n))
    _, cts = _vital_inputs(P, keys, cfg, 3, 3102)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    N, D = cc.vitals_v1(ev, book, cts[0::2], cts[1::2], cfg)
    ctx = _run(m, P, keys, book, "vitals_v1", cfg, cts, [N, D])
    assert ctx.trace() == ev.trace
    assert sorted(ctx.required_rotations("vitals_v1", _mcfg(m, cfg))) == cc.required_rotations("vitals_v1", cfg, P.n)


def test_graph_replay_matches_eager(m):
    """Repeated device-resident eval_chain calls (trace off) are captured once and replayed
    as a CUDA graph: residues stay bit-exact with the oracle on every call, the launch
    count per call is unchanged, replays re-read new input contents, and an operand-store
    change invalidates the captured graph."""
    import torch
    P = toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)
    cfg = cc.ChainCfg(R=16, F=6, gamma=2, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=3151, rotations=cc.required_rotations("vitals_v1", cfg, P.n))
    book = cc.PlainBook(P)
    wants = []
    inputs = []
    for seed in (3152, 3153):
        _, cts = _vital_inputs(P, keys, cfg, 3, seed)
        ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
        wants.append(cc.vitals_v1(ev, book, cts[0::2], cts[1::2], cfg))
        inputs.append(cts)
    ctx = make_ctx(m, P, keys, book)
    ctx.trace_enable(False)
    mcfg = _mcfg(m, cfg)
    ins = [ct_in(m, P, c) for c in inputs[0]]
    outs = [ct_out(m, P, lv) for lv in ctx.chain_plan("vitals_v1", mcfg, 3, len(ins))]

    def check(want):
        for o, w in zip(outs, want):
            assert np.array_equal(residues(o), np.stack(w.c))
            assert o.level == w.level and o.scale == w.scale

    deltas = []
    for _ in range(4):
        l0 = ctx.launch_count()
        ctx.eval_chain("vitals_v1", mcfg, ins, outs)
        torch.cuda.synchronize()
        deltas.append(ctx.launch_count() - l0)
        check(wants[0])
    assert len(set(deltas)) == 1 and deltas[0] > 0
    n_graphs, replays = ctx.graph_stats()
    assert n_graphs == 1 and replays == 3  # call 2 captured + launched, calls 3-4 replayed
    # same buffers, new contents: the replay reads them
    for x, c in zip(ins, inputs[1]):
        x.data.copy_(ct_in(m, P, c).data)
    ctx.eval_chain("vitals_v1", mcfg, ins, outs)
    torch.cuda.synchronize()
    assert ctx.graph_stats()[1] == 4
    check(wants[1])
    # an operand-store change drops the graphs; the next call runs eagerly and is still exact
    ctx.load_scalars("unused", [1.0])
    assert ctx.graph_stats()[0] == 0
    for o in outs:
        o.data.zero_()
    ctx.eval_chain("vitals_v1", mcfg, ins, outs)
    torch.cuda.synchronize()
    check(wants[1])
    # graphs off: eager every call
    ctx.graph_enable(False)
    ctx.eval_chain("vitals_v1", mcfg, ins, outs)
    ctx.eval_chain("vitals_v1", mcfg, ins, outs)
    torch.cuda.synchronize()
    assert ctx.graph_stats() == (0, 4)
    check(wants[1])


def test_eval_chain_async_host_buffers(m):
    """mmfhe_eval_chain_async with pinned host buffers: several calls in flight (two
    staging slots, graph replay after warm-up), alternating input sets into separate
    output buffers, read after sync(): every output bit-exact with the oracle."""
    import torch
    P = toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)
    cfg = cc.ChainCfg(R=16, F=6, gamma=2, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=3161, rotations=cc.required_rotations("vitals_v1", cfg, P.n))
    book = cc.PlainBook(P)
    wants, hins = [], []
    for seed in (3162, 3163):
        _, cts = _vital_inputs(P, keys, cfg, 3, seed)
        ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
        wants.append(cc.vitals_v1(ev, book, cts[0::2], cts[1::2], cfg))
        data = torch.from_numpy(np.stack([np.stack(c.c) for c in cts]).view(np.int64)).pin_memory()
        hins.append(m.CtArray([m.Ct(data[i], 3, cts[i].scale, cts[i].n_slots, P.log_n, m.FORM_COEFF, 2)
                               for i in range(len(cts))]))
    ctx = make_ctx(m, P, keys, book)
    ctx.trace_enable(False)
    mcfg = _mcfg(m, cfg)
    levels = ctx.chain_plan("vitals_v1", mcfg, 3, len(hins[0]))
    calls = []
    for it in range(6):
        outs = [m.Ct(torch.empty((2, lv + 1, P.n), dtype=torch.int64).pin_memory(), lv, 0.0, 0, P.log_n)
                for lv in levels]
        arr = m.CtArray(outs)
        ctx.eval_chain_async("vitals_v1", mcfg, hins[it % 2], arr)
        calls.append((it % 2, outs, arr))
    ctx.sync()
    for which, outs, arr in calls:
        for o, w in zip(outs, wants[which]):
            assert np.array_equal(residues(o), np.stack(w.c))
            assert o.level == w.level and o.scale == w.scale
    assert ctx.graph_stats()[1] >= 2  # both staging slots reached graph replay


def _gesture(P, seed, F=2, A=2, R=4, D=8, frame_batch=0, hoist=0):
    n = A * R * D
    cfg = cc.ChainCfg(A=A, R=R, D=D, F=F, gamma=4, n_slots=n, fc_dims=(n, 16, 8, 8), frame_batch=frame_batch,
                      hoist=hoist)
    Z, _ = radar.gesture_scene(A, R, D, F, seed=seed, cls=seed % 5)
    return cfg, radar.preprocess_gesture(Z)


@pytest.mark.parametrize("F,fb,hoist", [(2, 0, 0), (3, 2, 0), (3, 2, 1)])
def test_gesture_chain_small(m, F, fb, hoist):
    P = toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)
    cfg, Zt = _gesture(P, 3201, F=F, frame_batch=fb, hoist=hoist)
    keys = orc.keygen(P, seed=3202, rotations=cc.required_rotations("gesture", cfg, P.n))
    cts = []
    for t in range(cfg.F):
        v = radar.pack_doppler(Zt[t])
        for part in (v.real, v.imag):
            cts.append(orc.encrypt_vector(P, keys, part, P.L, seed=3203, index=len(cts)))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    feat = cc.gesture_features(ev, book, cts[0::2], cts[1::2], cfg)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=3204)
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    ctx = _run(m, P, keys, book, "gesture", cfg, cts, [logits])
    assert ctx.trace() == ev.trace
    assert sorted(ctx.required_rotations("gesture", _mcfg(m, cfg))) == cc.required_rotations("gesture", cfg, P.n)
    # per-frame chain and FC chain on their own
    ev2 = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    f0 = cc.gesture_frame(ev2, cc.PlainBook(P), cts[0], cts[1], cfg)
    _run(m, P, keys, book, "gesture_frame", cfg, cts[:2], [f0])


@pytest.mark.parametrize("lanes,F,fb,hoist,merge", [(4, 6, 0, 1, 0), (2, 5, 2, 1, 0), (8, 8, 0, 1, 0), (4, 6, 0, 2, 0),
                                                    (2, 5, 2, 2, 0), (1, 3, 2, 2, 0), (2, 5, 2, 2, 1), (1, 3, 2, 2, 1)])
def test_gesture_chain_lanes_small(m, lanes, F, fb, hoist, merge):
    """SIMD-dense gesture pipeline (DESIGN R20): `lanes` frames interleaved per ciphertext,
    ceil(F / lanes) ciphertext pairs (the last one partly empty), hoisted (hoist = 1) or
    double-hoisted (hoist = 2: PQ baby steps, PQ diagonals, PQ giant steps, one ModDown per
    output) BSGS in K3 and the FC head with the lane sum: residues and trace equal the
    oracle's; K3 alone too."""
    P = toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)
    cfg, Zt = _gesture(P, 3221, F=F, frame_batch=fb, hoist=hoist)
    cfg.lanes, cfg.ks_merge = lanes, merge  # merge: relin / ModDown + rescale as one division (R31)
    keys = orc.keygen(P, seed=3222, rotations=cc.required_rotations("gesture", cfg, P.n))
    n = cfg.n_slots
    cts = []
    vs = [radar.pack_doppler(Zt[t]) for t in range(F)]
    for g in range(cc.n_packed(F, lanes)):
        grp = vs[g * lanes:(g + 1) * lanes]
        for part in ("real", "imag"):
            cts.append(orc.encrypt_vector(P, keys, cc.interleave([getattr(v, part) for v in grp], lanes, n), P.L,
                                          seed=3223, index=len(cts)))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    feat = cc.gesture_features(ev, book, cts[0::2], cts[1::2], cfg)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=3224)
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    ctx = _run(m, P, keys, book, "gesture", cfg, cts, [logits])
    assert ctx.trace() == ev.trace
    assert sorted(ctx.required_rotations("gesture", _mcfg(m, cfg))) == cc.required_rotations("gesture", cfg, P.n)
    ev2 = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book2 = cc.PlainBook(P)
    dre, dim = cc.k3_doppler_dft_frames(ev2, book2, cts[0:2:2], cts[1:2:2], cfg)
    _run(m, P, keys, book2, "k3_doppler_dft", cfg, cts[:2], dre + dim)


@pytest.mark.parametrize("lanes,F,fb,hoist,aligned", [(1, 2, 0, 0, 0), (1, 3, 2, 1, 0), (2, 5, 2, 2, 0), (4, 6, 0, 2, 0),
                                                      (1, 2, 0, 0, 1), (2, 5, 2, 2, 1), (4, 6, 0, 2, 1),
                                                      (1, 6, 0, 2, 1), (4, 6, 0, 2, 2), (2, 5, 2, 2, 3),
                                                      (4, 6, 0, 2, 4), (1, 3, 0, 2, 5), (4, 6, 0, 2, 6),
                                                      (1, 6, 0, 2, 6), (4, 6, 0, 2, 7), (1, 3, 0, 2, 7),
                                                      (1, 3, 0, 2, 8)])
def test_gesture_chain_complex_small(m, lanes, F, fb, hoist, aligned):
    """Complex-slot gesture pipeline (cfg.cplx, DESIGN R28): one ciphertext z = v_re + j v_im
    per frame group, K3 with complex diagonals (one plaintext product per diagonal), K1 as
    d Conj(d) with the conjugation key: residues and trace equal the oracle's for the whole
    chain, and for K3 and the per-frame chain on their own; the required key set ends with
    the conjugation key id."""
    P = toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)
    cfg, Zt = _gesture(P, 3241, F=F, frame_batch=fb, hoist=hoist)
    # aligned 2 / 3: the aligned schedule with a double-hoisted rotate-and-sum level of 16 / 4 (R27);
    # 4 / 5: every level hoisted in groups of 2 / 4 (R30)
    cfg.lanes, cfg.cplx, cfg.bsgs_aligned = lanes, 1, min(aligned, 1)
    cfg.rotsum_inner = {2: 16, 3: 4, 4: 2, 5: 4}.get(aligned, 0)
    cfg.rotsum_hoist_all = int(aligned >= 4)
    cfg.ks_merge = int(aligned >= 6)  # 6: + relin / ModDown + rescale as one division (R31)
    cfg.k1_conj_fuse = int(aligned >= 7)  # 7: + K1 as one conjugate-product key switch (R32)
    if aligned == 8:  # 8: 20 baby steps (> 16): the 32-wide staged diagonal MAC with its split sum
        cfg.bsgs_baby = 20
    if aligned == 6:
        cfg.rotsum_inner = 2
    rots = cc.required_rotations("gesture", cfg, P.n)
    assert rots[0] == orc.CONJ == m.STEP_CONJ
    assert (orc.CONJ_PROD in rots) == bool(cfg.k1_conj_fuse) and orc.CONJ_PROD == m.STEP_CONJ_PROD
    keys = orc.keygen(P, seed=3242, rotations=rots)
    n = cfg.n_slots
    vs = [radar.pack_doppler(Zt[t]) for t in range(F)]
    cts = [orc.encrypt_vector(P, keys, cc.interleave(vs[g * lanes:(g + 1) * lanes], lanes, n), P.L, seed=3243, index=g)
           for g in range(cc.n_packed(F, lanes))]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    feat = cc.gesture_features(ev, book, cts, None, cfg)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=3244)
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    ctx = _run(m, P, keys, book, "gesture", cfg, cts, [logits])
    assert ctx.trace() == ev.trace
    assert (("conj_mul_relin_rescale" if cfg.k1_conj_fuse else "conj"), P.L - 1, "") in ev.trace
    assert sorted(ctx.required_rotations("gesture", _mcfg(m, cfg))) == rots
    ev2 = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book2 = cc.PlainBook(P)
    d = cc.k3_doppler_dft_frames_c(ev2, book2, cts[:1], cfg)
    c2 = _run(m, P, keys, book2, "k3_doppler_dft", cfg, cts[:1], d)
    assert c2.trace() == ev2.trace
    ev3 = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book3 = cc.PlainBook(P)
    f0 = cc.gesture_frame(ev3, book3, cts[0], None, cfg)
    _run(m, P, keys, book3, "gesture_frame", cfg, cts[:1], [f0])
    # the split layout's input count is rejected for complex slots, and vice versa
    with pytest.raises(m.MmfheError):
        ctx.chain_plan("gesture", _mcfg(m, cfg), P.L, 2 * len(cts))
    # without the conjugation key the chain stops with E_MISSING_KEY naming that key
    nokey = orc.Keys(keys.s, keys.pk, keys.rlk, {k: v for k, v in keys.gk.items() if k != orc.CONJ})
    ctx3 = make_ctx(m, P, nokey, book)
    with pytest.raises(m.MmfheError) as e:
        ctx3.eval_chain("gesture", _mcfg(m, cfg), [ct_in(m, P, c) for c in cts], [ct_out(m, P, logits.level)])
    assert e.value.name == "E_MISSING_KEY" and "conjugation" in str(e.value)


@pytest.mark.parametrize("cplx", [0, 1])
def test_gesture_features_sessions_batched(m, cplx):
    """gesture_features over S = 3 sessions in one call (cfg.sessions): every session's frame
    groups run as one batch through the per-frame chain and each session's frames are summed on
    their own; output s equals the oracle's gesture_features of session s alone, residue for
    residue (split re / im layout, and complex slots with the headline's R27-R32 options)."""
    P = toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)
    S, F, lanes = 3, 4, 2
    cfg, _ = _gesture(P, 3251, F=F, hoist=2)
    cfg.lanes, cfg.cplx = lanes, cplx
    if cplx:
        cfg.bsgs_aligned, cfg.rotsum_inner, cfg.rotsum_hoist_all, cfg.ks_merge, cfg.k1_conj_fuse = 1, 4, 1, 1, 1
    keys = orc.keygen(P, seed=3252, rotations=cc.required_rotations("gesture_features", cfg, P.n))
    n = cfg.n_slots
    book = cc.PlainBook(P)
    ins, want = [], []
    for s in range(S):
        _, Zt = _gesture(P, 3260 + s, F=F)
        vs = [radar.pack_doppler(Zt[t]) for t in range(F)]
        groups = [vs[g * lanes:(g + 1) * lanes] for g in range(cc.n_packed(F, lanes))]
        ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
        if cplx:
            cts = [orc.encrypt_vector(P, keys, cc.interleave(grp, lanes, n), P.L, seed=3270 + s, index=g)
                   for g, grp in enumerate(groups)]
            want.append(cc.gesture_features(ev, book, cts, None, cfg))
        else:
            cts = []
            for grp in groups:
                for part in ("real", "imag"):
                    cts.append(orc.encrypt_vector(P, keys, cc.interleave([getattr(v, part) for v in grp], lanes, n),
                                                  P.L, seed=3270 + s, index=len(cts)))
            want.append(cc.gesture_features(ev, book, cts[0::2], cts[1::2], cfg))
        ins += cts
    ctx = make_ctx(m, P, keys, book)
    mcfg = _mcfg(m, cfg)
    mcfg.sessions = S
    levels = ctx.chain_plan("gesture_features", mcfg, P.L, len(ins))
    assert levels == [w.level for w in want]
    outs = [ct_out(m, P, lv) for lv in levels]
    assert ctx.eval_chain("gesture_features", mcfg, [ct_in(m, P, c) for c in ins], outs) == S
    for o, w in zip(outs, want):
        assert np.array_equal(residues(o), np.stack(w.c)), "residues differ from the oracle"
        assert o.scale == w.scale and o.level == w.level
    # the inputs must split into equal runs, and only gesture_features takes sessions
    with pytest.raises(m.MmfheError):
        ctx.chain_plan("gesture_features", mcfg, P.L, len(ins) - (1 if cplx else 2))
    with pytest.raises(m.MmfheError):
        ctx.chain_plan("gesture", mcfg, P.L, len(ins))


def test_frame_sharded_gesture_exchange(m):
    """frames of one session split over 'ranks' (here 3 shards on one GPU),
    per-shard gesture_features, library sum of the partials, FC head -- equals the
    oracle's single-device gesture pipeline residue for residue (sums are exact mod q)."""
    from paper_2603_22437_b200.dist import shard
    P = toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)
    cfg, Zt = _gesture(P, 3211, F=5, frame_batch=2, hoist=1)
    keys = orc.keygen(P, seed=3212, rotations=cc.required_rotations("gesture", cfg, P.n))
    cts = []
    for t in range(cfg.F):
        v = radar.pack_doppler(Zt[t])
        for part in (v.real, v.imag):
            cts.append(orc.encrypt_vector(P, keys, part, P.L, seed=3213, index=len(cts)))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    feat = cc.gesture_features(ev, book, cts[0::2], cts[1::2], cfg)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=3214)
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    ctx = make_ctx(m, P, keys, book)
    mcfg = _mcfg(m, cfg)
    parts = []
    for r in range(3):
        lo, hi = shard(cfg.F, r, 3)
        o = ct_out(m, P, feat.level)
        ctx.eval_chain("gesture_features", mcfg, [ct_in(m, P, c) for c in cts[2 * lo:2 * hi]], [o])
        parts.append(o)
    total = ct_out(m, P, feat.level)
    ctx.sum_partials(parts, total)
    assert np.array_equal(residues(total), np.stack(feat.c)) and total.scale == feat.scale
    out = ct_out(m, P, logits.level)
    ctx.eval_chain("gesture_fc", mcfg, [total], [out])
    assert np.array_equal(residues(out), np.stack(logits.c))


def test_k3_doppler_dft_c3_full_size(m):
    """C3: block-diagonal Doppler DFT via slot rotations, N=2^15, A=4 x R=32 x D=32."""
    P = ps3()
    cfg = cc.ChainCfg(A=4, R=32, D=32, F=1, n_slots=4096)
    keys = orc.keygen(P, seed=3301, rotations=cc.required_rotations("k3_doppler_dft", cfg, P.n))
    Z, _ = radar.gesture_scene(4, 32, 32, 3, seed=3302, cls=2)
    Zt = radar.preprocess_gesture(Z)
    v = radar.pack_doppler(Zt[1])
    cre = orc.encrypt_vector(P, keys, v.real, P.L, seed=3303, index=0)
    cim = orc.encrypt_vector(P, keys, v.imag, P.L, seed=3303, index=1)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    dre, dim = cc.k3_doppler_dft(ev, book, cre, cim, cfg)
    ctx = _run(m, P, keys, book, "k3_doppler_dft", cfg, [cre, cim], [dre, dim])
    assert ctx.trace() == ev.trace
    assert sum(1 for op in ev.trace if op[0] == "hrot") == 30
    want = dsp.doppler_dft(v, cfg.D)
    got = orc.decrypt_vector(P, keys, dre)
    assert np.max(np.abs(got - want.real)) <= 1e-3 * np.max(np.abs(want.real))


@pytest.mark.parametrize("taps", [
    # linear-phase (symmetric) taps: the paired k_lincomb_sym path, even and odd length
    ([0.2, 0.3, 0.3, 0.2], [0.25, -0.5, 0.25]),
    # asymmetric taps: the general k_lincomb_mat path
    ([0.1, 0.3, 0.4, 0.2], [0.25, -0.5, 0.3]),
])
def test_vitals_v2_small(m, taps):
    P = toy(log_n=10, n_q=10, scale_bits=40, n_p=2, alpha=2)  # third order needs 9 levels
    cfg = cc.ChainCfg(R=8, F=10, p_phi=2, taylor_order=3, n_slots=P.n // 2, fs=2.0,
                      bands=((0.1, 0.6), (0.7, 1.0)), frame_batch=4)
    keys = orc.keygen(P, seed=3401, rotations=cc.required_rotations("vitals_v2", cfg, P.n))
    _, cts = _vital_inputs(P, keys, cfg, 9, 3402)
    taps = [np.array(t) for t in taps]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    out = cc.vitals_v2(ev, cts[0::2], cts[1::2], taps, cfg)
    want = out[0] + out[1]
    scalars = {f"k5.b{b}": t for b, t in enumerate(taps)}
    bins = []
    for b in range(2):
        ks = dsp.band_bins(cfg.F - 1, cfg.fs, cfg.bands[b])
        bins.append([int(k) for k in ks])
        for k in ks:
            c, s = dsp.narrowband_dft_coefs(cfg.F - 1, int(k))
            scalars[f"vp.c.{b}.{int(k)}"] = c
            scalars[f"vp.s.{b}.{int(k)}"] = s
    ctx = _run(m, P, keys, None, "vitals_v2", cfg, cts, want, scalars=scalars, bins=bins, taps=taps)
    assert ctx.trace() == ev.trace


@pytest.mark.parametrize("taps", [([0.2, 0.3, 0.3, 0.2], [0.25, -0.5, 0.25])])
@pytest.mark.parametrize("iq_pack,hoist", [(0, 0), (1, 0), (3, 0), (3, 1)])
def test_vitals_v2_vp_plus(m, taps, iq_pack, hoist):
    """Full-depth V2 (VP+ sharpen + weighted frequency average in the cloud):
    N_f, D_f residues and the op trace equal the oracle's."""
    P = toy(log_n=10, n_q=10, scale_bits=50, n_p=2, alpha=2)
    # iq_pack = 3 packs 4 frames: every frame batch a multiple of 4
    cfg = cc.ChainCfg(R=8, F=12 if iq_pack == 3 else 10, p_phi=2, taylor_order=1, n_slots=P.n // 2, fs=2.0,
                      bands=((0.1, 0.6), (0.7, 1.0)), frame_batch=4, vp_plus=1, iq_pack=iq_pack, hoist=hoist)
    keys = orc.keygen(P, seed=3501, rotations=cc.required_rotations("vitals_v2", cfg, P.n))
    _, cts = _vital_inputs(P, keys, cfg, 9, 3502)
    taps = [np.array(t) for t in taps]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    out = cc.vitals_v2(ev, cts[0::2], cts[1::2], taps, cfg)
    want = out[0] + out[1]
    assert len(want) == 4 and want[0].level == 0
    scalars = {f"k5.b{b}": t for b, t in enumerate(taps)}
    bins = []
    for b in range(2):
        ks = dsp.band_bins(cfg.F - 1, cfg.fs, cfg.bands[b])
        bins.append([int(k) for k in ks])
        for k in ks:
            c, s = dsp.narrowband_dft_coefs(cfg.F - 1, int(k))
            scalars[f"vp.c.{b}.{int(k)}"] = c
            scalars[f"vp.s.{b}.{int(k)}"] = s
    ctx = _run(m, P, keys, None, "vitals_v2", cfg, cts, want, scalars=scalars, bins=bins, taps=taps)
    assert ctx.trace() == ev.trace


@pytest.mark.parametrize("iq_pack,hoist,merge", [(0, 0, 0), (3, 1, 0), (3, 1, 1)])
def test_vital_sessions_packed(m, iq_pack, hoist, merge):
    """Vital sessions packed per ciphertext (DESIGN R33): S = N / (2 R 2^iq_pack) sessions in the slot
    blocks of every input ciphertext, cfg.n_slots = R 2^iq_pack; V1 and the full-depth V2 (VP+):
    residues and op traces equal the oracle's (whose per-session decryption is pinned against each
    session's DSP in test_oracle_circuits.py::test_vital_sessions_packed_per_ciphertext)."""
    P = toy(log_n=10, n_q=10, scale_bits=50, n_p=2, alpha=2)
    R, F = 8, 12
    n = R << iq_pack
    S = (P.n // 2) // n
    cfg = cc.ChainCfg(R=R, F=F, gamma=2, p_phi=2, taylor_order=1, n_slots=n, fs=2.0, bands=((0.1, 0.6), (0.7, 1.0)),
                      frame_batch=4, vp_plus=1, iq_pack=iq_pack, hoist=hoist, ks_merge=merge)
    scenes = [radar.preprocess_vital(radar.vital_scene(R, F, cfg.fs, seed=3600 + s)[0]) for s in range(S)]
    rots = sorted(set(cc.required_rotations("vitals_v1", cfg, P.n)) | set(cc.required_rotations("vitals_v2", cfg, P.n)))
    keys = orc.keygen(P, seed=3601, rotations=rots)

    def cts(lvl):
        out = []
        for t in range(F):
            for part in ("real", "imag"):
                v = np.concatenate([radar.pack_vital(getattr(scenes[s][t], part), n) for s in range(S)])
                sc = float(2 ** P.scale_bits)
                out.append(orc.encrypt(P, keys, orc.encode(P, v, sc, lvl), lvl, sc, n, seed=3602, index=len(out)))
        return out

    c1 = cts(3)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    Nc, Dc = cc.vitals_v1(ev, book, c1[0::2], c1[1::2], cfg)
    ctx = _run(m, P, keys, book, "vitals_v1", cfg, c1, [Nc, Dc])
    assert ctx.trace() == ev.trace
    c2 = cts(9)
    taps = [np.array([0.2, 0.3, 0.3, 0.2]), np.array([0.25, -0.5, 0.25])]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    out = cc.vitals_v2(ev, c2[0::2], c2[1::2], taps, cfg)
    scalars = {f"k5.b{b}": t for b, t in enumerate(taps)}
    bins = []
    for b in range(2):
        ks = dsp.band_bins(F - 1, cfg.fs, cfg.bands[b])
        bins.append([int(k) for k in ks])
        for k in ks:
            c, s_ = dsp.narrowband_dft_coefs(F - 1, int(k))
            scalars[f"vp.c.{b}.{int(k)}"] = c
            scalars[f"vp.s.{b}.{int(k)}"] = s_
    ctx = _run(m, P, keys, None, "vitals_v2", cfg, c2, out[0] + out[1], scalars=scalars, bins=bins, taps=taps)
    assert ctx.trace() == ev.trace


def test_chain_shape_and_depth_errors(m):
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    ctx = make_ctx(m, P)
    cfg = _mcfg(m, cc.ChainCfg(R=8, F=3, gamma=2, n_slots=P.n // 2))
    with pytest.raises(m.MmfheError) as e:
        ctx.chain_plan("vitals_v1", cfg, 3, 5)
    assert e.value.name == "E_SHAPE"
    with pytest.raises(m.MmfheError) as e:
        ctx.chain_plan("vitals_v1", cfg, 2, 6)
    assert e.value.name == "E_DEPTH"
    with pytest.raises(m.MmfheError) as e:
        ctx.chain_plan("no_such_chain", cfg, 3, 6)
    assert e.value.name == "E_INVALID_ARG"
    # packed K4 rotate-and-sum (R19): frame batches must hold whole packing groups, and the
    # client is told every key the packing needs
    bins = [[1], [2]]
    P8 = toy(log_n=10, n_q=8, scale_bits=40, n_p=2, alpha=2)
    ctx8 = make_ctx(m, P8)
    c3 = m.chain_cfg(R=8, F=6, p_phi=2, n_slots=P.n // 2, bands_bins=bins, n_taps=[3, 3], fs=2.0, iq_pack=3)
    with pytest.raises(m.MmfheError) as e:
        ctx8.chain_plan("vitals_v2", c3, 7, 12)
    assert e.value.name == "E_SHAPE"
    c3 = m.chain_cfg(R=8, F=8, p_phi=2, n_slots=P.n // 2, bands_bins=bins, n_taps=[3, 3], fs=2.0, iq_pack=3)
    assert len(ctx8.chain_plan("vitals_v2", c3, 7, 16)) == 2
    rots = ctx.required_rotations("vitals_v2", c3)
    assert all((8 << j) in rots and (P.n // 2 - (8 << j)) in rots for j in range(3))
    assert rots == cc.required_rotations("vitals_v2", cc.ChainCfg(R=8, F=8, n_slots=P.n // 2, iq_pack=3), P.n)
    # round-2 cfg fields (R27-R29): invalid values and chains they do not apply to are rejected
    g = dict(A=2, R=4, D=8, F=2, gamma=4, n_slots=64, fc_dims=(64, 16, 8, 8), hoist=2)
    ctx12 = make_ctx(m, toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2))
    for bad, name in ((dict(cplx=2), "E_INVALID_ARG"), (dict(bsgs_aligned=2), "E_INVALID_ARG"),
                      (dict(rotsum_inner=3), "E_INVALID_ARG"), (dict(rotsum_inner=128), "E_INVALID_ARG")):
        with pytest.raises(m.MmfheError) as e:
            ctx12.chain_plan("gesture", m.chain_cfg(**g, **bad), 11, 4)
        assert e.value.name == name, bad
    with pytest.raises(m.MmfheError) as e:
        ctx8.chain_plan("vitals_v1", m.chain_cfg(R=8, F=3, gamma=2, n_slots=P.n // 2, cplx=1), 3, 6)
    assert e.value.name == "E_SHAPE"
    # complex slots: one input per frame group, and the conjugation key is required
    cc_ = m.chain_cfg(**g, cplx=1)
    assert len(ctx12.chain_plan("gesture", cc_, 11, 2)) == 1
    with pytest.raises(m.MmfheError) as e:
        ctx12.chain_plan("gesture", cc_, 11, 4)
    assert e.value.name == "E_SHAPE"
    assert ctx12.required_rotations("gesture", cc_)[0] == m.STEP_CONJ
    assert m.STEP_CONJ not in ctx12.required_rotations("gesture", m.chain_cfg(**g))


# ------------------------------------------------------------------ the kernels on their own

def _enc_list(P, keys, vals, level, seed):
    return [orc.encrypt_vector(P, keys, v, level, seed=seed, index=i) for i, v in enumerate(vals)]


def test_standalone_k2_k4_k7_chains(m):
    """k2_soft_attention, k4_soft_iq (canonical and packed), k7_taylor_phase (first and
    third order) as chains of their own: residues and trace equal the oracle kernels'."""
    P = toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)
    rng = np.random.default_rng(71)
    cfg = cc.ChainCfg(R=8, F=8, gamma=2, p_phi=2, n_slots=P.n // 2, frame_batch=4)
    cfgp = cc.ChainCfg(R=8, F=8, gamma=2, p_phi=2, n_slots=P.n // 2, frame_batch=4, iq_pack=3, hoist=1)
    rots = sorted(set(cc.required_rotations("k2_soft_attention", cfg, P.n)) |
                  set(cc.required_rotations("k4_soft_iq", cfgp, P.n)))
    keys = orc.keygen(P, seed=3601, rotations=rots)
    # K2a on an energy ciphertext E (values in [0, F] in the first R slots)
    E = orc.encrypt_vector(P, keys, radar.pack_vital(rng.uniform(0, 8, 8), cfg.n_slots), 3, seed=3602, index=0)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    N, D = cc.k2_soft_attention(ev, book, E, cfg)
    ctx = _run(m, P, keys, book, "k2_soft_attention", cfg, [E], [N, D])
    assert ctx.trace() == ev.trace
    # K4 per frame batch (frame_batch 4), outputs I_0..I_{F-1}, Q_0..Q_{F-1}
    z = rng.uniform(-0.5, 0.5, (8, 8)) + 1j * rng.uniform(-0.5, 0.5, (8, 8))
    cts = []
    for t in range(8):
        for part in (z[t].real, z[t].imag):
            cts.append(orc.encrypt_vector(P, keys, radar.pack_vital(part, cfg.n_slots), 4, seed=3603,
                                          index=len(cts)))
    for c in (cfg, cfgp):
        ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
        I, Q = [], []
        for s, e in cc.chunks(8, c.frame_batch):
            Ib, Qb = cc.k4_soft_iq(ev, cts[2 * s:2 * e:2], cts[2 * s + 1:2 * e:2], c)
            I += Ib
            Q += Qb
        ctx = _run(m, P, keys, None, "k4_soft_iq", c, cts, I + Q)
        assert ctx.trace() == ev.trace
    # K7 on (I_f, Q_f) pairs
    P7 = toy(log_n=10, n_q=5, scale_bits=40, n_p=2, alpha=2)
    keys7 = orc.keygen(P7, seed=3604)
    th = np.cumsum(rng.uniform(-0.4, 0.4, (5, P7.n // 2)), axis=0)
    If = _enc_list(P7, keys7, np.cos(th), 4, 3605)
    Qf = _enc_list(P7, keys7, np.sin(th), 4, 3606)
    pairs = [x for t in range(5) for x in (If[t], Qf[t])]
    for order in (1, 3):
        c7 = cc.ChainCfg(taylor_order=order, n_slots=P7.n // 2)
        ev = cc.CircuitEvaluator(P7, keys7.rlk, keys7.gk)
        ys = cc.k7_taylor_phase(ev, If, Qf, order)
        ctx = _run(m, P7, keys7, None, "k7_taylor_phase", c7, pairs, ys)
        assert ctx.trace() == ev.trace


def test_standalone_k5_fir_long_window(m):
    """k5_fir on its own with an asymmetric 300-tap filter over 300 frames (the general
    k_lincomb_mat path, window > 256: the 128-bit accumulator's hi-word fold)
    and a symmetric 41-tap band (k_lincomb_sym): two bands, outputs band-major."""
    P = toy(log_n=10, n_q=3, scale_bits=40, n_p=1, alpha=1)
    rng = np.random.default_rng(72)
    F = 300
    keys = orc.keygen(P, seed=3611)
    xs = _enc_list(P, keys, rng.uniform(-1, 1, (F, P.n // 2)), 2, 3612)
    taps = [rng.uniform(-1, 1, 300), radar.fir_taps(41, (0.8, 2.5), 20.0)]
    cfg = cc.ChainCfg(F=F, n_slots=P.n // 2)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    want = []
    for h in taps:
        want += cc.k5_fir(ev, xs, h)
    scalars = {f"k5.b{b}": t for b, t in enumerate(taps)}
    ctx = _run(m, P, keys, None, "k5_fir", cfg, xs, want, scalars=scalars, bins=([1], [1]), taps=taps)
    assert ctx.trace() == ev.trace


@pytest.mark.parametrize("lanes", [1, 4])
def test_standalone_k6_k2b_fc_chains(m, lanes):
    """k6_notch, k2_doppler_soft_power and fc_forward as chains of their own (with and
    without SIMD-dense lanes): residues and trace equal the oracle kernels'."""
    P = toy(log_n=10, n_q=8, scale_bits=40, n_p=2, alpha=2)
    n = 64
    cfg = cc.ChainCfg(A=2, R=4, D=8, gamma=4, n_slots=n, fc_dims=(n, 16, 8, 8), hoist=1, lanes=lanes)
    rots = sorted(set(cc.required_rotations("k2_doppler_soft_power", cfg, P.n)) |
                  set(cc.required_rotations("fc_forward", cfg, P.n)))
    keys = orc.keygen(P, seed=3621, rotations=rots)
    rng = np.random.default_rng(73)
    vals = [cc.interleave([rng.uniform(0, 1, n) for _ in range(lanes)], lanes, n) for _ in range(3)]
    Ps = _enc_list(P, keys, vals, 7, 3622)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    want = cc.k6_notch(ev, book, Ps, cfg)
    ctx = _run(m, P, keys, book, "k6_notch", cfg, Ps, want)
    assert ctx.trace() == ev.trace
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    want = cc.k2_doppler_soft_power(ev, Ps, cfg)
    ctx = _run(m, P, keys, None, "k2_doppler_soft_power", cfg, Ps, want)
    assert ctx.trace() == ev.trace
    feat = Ps[0]
    Ws, bs = radar.fc_weights([n, 16, 8, 5], seed=3623)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    logits = cc.gesture_fc(ev, book, orc.Ct([c[:6].copy() for c in feat.c], 5, feat.scale, feat.n_slots),
                           Ws, bs, cfg)
    feat5 = orc.Ct([c[:6].copy() for c in feat.c], 5, feat.scale, feat.n_slots)
    ctx = _run(m, P, keys, book, "fc_forward", cfg, [feat5], [logits])
    assert ctx.trace() == ev.trace


@pytest.mark.parametrize("lanes,mode,S", [(1, 0, 3), (4, 0, 3), (4, 1, 3), (1, 1, 18)])
def test_fc_forward_sessions_batched(m, lanes, mode, S):
    """gesture_fc / fc_forward over several sessions' features in one call (the sessions as one
    batch, every op one launch): output s equals the oracle's gesture_fc of session s alone,
    residue for residue.  mode 1 is the bench's head configuration (double-hoisted BSGS, every
    rotate-and-sum level hoisted in groups of 4, merged divisions, R27 / R30 / R31); S = 18
    runs the grouped hoisted inner product in balanced batch chunks (6 + 6 + 6)."""
    P = toy(log_n=10, n_q=8, scale_bits=40, n_p=2, alpha=2)
    n = 64
    cfg = cc.ChainCfg(A=2, R=4, D=8, gamma=4, n_slots=n, fc_dims=(n, 16, 8, 8), hoist=1 + mode, lanes=lanes)
    if mode:
        cfg.rotsum_inner, cfg.rotsum_hoist_all, cfg.ks_merge = 4, 1, 1
    keys = orc.keygen(P, seed=3625, rotations=cc.required_rotations("fc_forward", cfg, P.n))
    rng = np.random.default_rng(75)
    vals = [cc.interleave([rng.uniform(0, 1, n) for _ in range(lanes)], lanes, n) for _ in range(S)]
    feats = [orc.Ct([c[:6].copy() for c in f.c], 5, f.scale, f.n_slots) for f in _enc_list(P, keys, vals, 7, 3626)]
    Ws, bs = radar.fc_weights([n, 16, 8, 5], seed=3627)
    book = cc.PlainBook(P)
    want = [cc.gesture_fc(cc.CircuitEvaluator(P, keys.rlk, keys.gk), book, f, Ws, bs, cfg) for f in feats]
    _run(m, P, keys, book, "fc_forward", cfg, feats, want)
    _run(m, P, keys, book, "gesture_fc", cfg, feats[:2], want[:2])


@pytest.mark.parametrize("hoist", [0, 1])
def test_standalone_k5_fir_rot(m, hoist):
    """The rotation-based FIR as a chain: two slot-packed sequences, a 41-tap and a
    5-tap band (BSGS over the taps, exact scalar combinations, hoisted or plain baby steps):
    residues and trace equal the oracle's k5_fir_rot, outputs band-major."""
    P = toy(log_n=10, n_q=3, scale_bits=40, n_p=2, alpha=2)
    rng = np.random.default_rng(74)
    F = 100
    taps = [radar.fir_taps(41, (0.8, 2.5), 20.0), radar.fir_taps(5, (0.1, 0.6), 20.0)]
    cfg = cc.ChainCfg(F=F, n_slots=P.n // 2, n_taps=(41, 5), hoist=hoist)
    keys = orc.keygen(P, seed=3631, rotations=cc.required_rotations("k5_fir_rot", cfg, P.n))
    seqs = []
    for _ in range(2):
        x = np.zeros(P.n // 2)
        x[:F] = rng.uniform(-1, 1, F)
        seqs.append(x)
    xs = _enc_list(P, keys, seqs, 2, 3632)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    want = [cc.k5_fir_rot(ev, x, h, hoist) for h in taps for x in xs]
    scalars = {f"k5.b{b}": t for b, t in enumerate(taps)}
    ctx = _run(m, P, keys, None, "k5_fir_rot", cfg, xs, want, scalars=scalars, bins=([1], [1]), taps=taps)
    assert ctx.trace() == ev.trace
    assert sorted(ctx.required_rotations("k5_fir_rot", _mcfg(m, cfg, bins=([1], [1]), taps=taps))) == \
        cc.required_rotations("k5_fir_rot", cfg, P.n)


def test_raw_adc_range_fft_then_vitals_v1(m):
    """The paper's raw-ADC variant: the encrypted range FFT of
    raw complex ADC samples by the K3 kernel (block DFT over the M samples of a chirp, Eq.
    range_fft P:1634-1640, windowed and fftshifted), composed with vitals_v1 on the K3
    outputs: residues and traces equal the oracle's; the decrypted soft-argmax bin equals
    the plaintext one computed from numpy's FFT of the same samples."""
    P = toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)
    M, F = 16, 6
    x, truth = radar.vital_adc_scene(M, F, 20.0, seed=3701)
    xt = radar.preprocess_adc(x)
    # one chirp of M samples in the first M slots of a period-2M vector (K3's Halevi-Shoup
    # diagonals over [-(D-1), D-1] need at least two blocks per period); block 1 stays zero
    cfg3 = cc.ChainCfg(A=1, R=2, D=M, n_slots=2 * M, hoist=1)
    cfg1 = cc.ChainCfg(R=M, F=F, gamma=2, n_slots=2 * M)
    rots = sorted(set(cc.required_rotations("k3_doppler_dft", cfg3, P.n)) |
                  set(cc.required_rotations("vitals_v1", cfg1, P.n)))
    keys = orc.keygen(P, seed=3702, rotations=rots)
    cts = []
    for t in range(F):
        for part in (xt[t].real, xt[t].imag):
            cts.append(orc.encrypt_vector(P, keys, radar.pack_vital(part, 2 * M), P.L, seed=3703, index=len(cts)))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    dre, dim = cc.k3_doppler_dft_frames(ev, book, cts[0::2], cts[1::2], cfg3)
    ctx = _run(m, P, keys, book, "k3_doppler_dft", cfg3, cts, dre + dim)
    assert ctx.trace() == ev.trace
    spec = [c for t in range(F) for c in (dre[t], dim[t])]
    ev1 = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book1 = cc.PlainBook(P)
    N, D = cc.vitals_v1(ev1, book1, spec[0::2], spec[1::2], cfg1)
    ctx1 = _run(m, P, keys, book1, "vitals_v1", cfg1, spec, [N, D])
    assert ctx1.trace() == ev1.trace
    X = np.fft.fftshift(np.fft.fft(np.hanning(M) * xt, axis=1), axes=1)
    got = orc.decrypt_vector(P, keys, dre[0])
    assert np.max(np.abs(got[:M] - X[0].real)) <= 1e-3 * np.max(np.abs(X[0].real))
    assert np.max(np.abs(got[M:])) <= 1e-6
    _, _, r_plain = dsp.soft_attention(dsp.energy(X), 2, F)
    r_enc = orc.decrypt_vector(P, keys, N)[0] / orc.decrypt_vector(P, keys, D)[0]
    assert round(r_enc) == round(r_plain)
    assert abs(round(r_plain) - (truth["r_star"] + M // 2) % M) <= 1
