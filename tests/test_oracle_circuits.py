"""Pins for the oracle's kernel circuits.

* schedule checks on plaintext slot vectors (BSGS K3, hybrid-diagonal FC):
  written with numpy rolls, compared with the plain matrix products;
* the DFT matrix of Eq. dft_kernel against numpy's fftshift(fft(w x));
* encrypted chains (O-RNS) decrypted and compared with O-DSP closed forms at
  the north-star gate: normwise 1e-3 relative;
* data obliviousness (Theorem P:999-1006): identical op traces on different
  inputs.
"""
import json
import os

import numpy as np
import pytest

from oracle import ckks as orc
from oracle import circuits as cc
from oracle import dsp
from synth import radar
from synth.params import toy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel_err(got, want):
    return float(np.max(np.abs(np.asarray(got) - np.asarray(want))) / max(np.max(np.abs(want)), 1e-300))


def test_dft_matrix_is_shifted_windowed_fft():
    D = 32
    rng = np.random.default_rng(0)
    x = rng.normal(size=D) + 1j * rng.normal(size=D)
    W = dsp.dft_matrix(D)
    want = np.fft.fftshift(np.fft.fft(np.hanning(D) * x))
    assert np.allclose(W @ x, want, atol=1e-12)


@pytest.mark.parametrize("D,b,aligned", [(8, 0, 0), (32, 0, 0), (32, 4, 0), (16, 5, 0), (8, 0, 1), (32, 0, 1),
                                         (32, 16, 1), (16, 5, 1), (32, 7, 1)])
def test_k3_bsgs_schedule_on_plain_slots(D, b, aligned):
    """The BSGS schedule (pre-rotated diagonals, babies, giants) reproduces the
    block-diagonal matvec exactly on plaintext slot vectors -- the SURVEY §8(c)-7 split and
    the aligned one (R29: giants at multiples of b, one of them the identity)."""
    n = 4 * D
    cfg = cc.ChainCfg(D=D, bsgs_baby=b, bsgs_aligned=aligned)
    rng = np.random.default_rng(D + b)
    M = rng.normal(size=(D, D))
    x = rng.normal(size=n)
    bb, giants = cc.k3_schedule(cfg)
    babies = [cc.rot(x, s) for s in range(bb)]
    y = np.zeros(n)
    n_rot = bb - 1
    for gp, G, ss in giants:
        inner = sum(cc.rot(cc.block_diag_diagonal(M, n, G + s), -G) * babies[s] for s in ss)
        y += cc.rot(inner, G)
        n_rot += G != 0
    want = (np.kron(np.eye(n // D), M) @ x)
    assert np.allclose(y, want)
    # 2D-1 nonzero diagonals; ~2 sqrt(d) rotations per input
    assert sum(len(ss) for _, _, ss in giants) == 2 * D - 1
    if D == 32 and b == 0:
        # 7 baby + 8 giant; x2 inputs -> 30 HRots per frame (aligned: 7 + 7, the giant G = 0 is free)
        assert n_rot == (14 if aligned else 15)
    if aligned:
        assert [G for _, G, _ in giants].count(0) == 1 and all(G % bb == 0 for _, G, _ in giants)
    if D == 32 and b == 16:
        assert n_rot == 15 + 3  # the headline's K3 split: 15 baby steps, 3 giant rotations


@pytest.mark.parametrize("h,n_in", [(8, 64), (16, 64), (5, 40)])
def test_fc_hybrid_diagonal_on_plain_slots(h, n_in):
    rng = np.random.default_rng(h)
    W = rng.normal(size=(h, n_in))
    x = rng.normal(size=n_in)
    b, giants = cc.fc_schedule(h)
    babies = [cc.rot(x, s) for s in range(b)]
    z = np.zeros(n_in)
    for gp, G, ss in giants:
        z += cc.rot(sum(cc.rot(cc.fc_diagonal(W, n_in, G + s), -G) * babies[s] for s in ss), G)
    if n_in % h == 0:
        y = sum(cc.rot(z, c * h) for c in range(n_in // h))
        assert np.allclose(y[:h], W @ x)
        assert np.allclose(y, np.tile(W @ x, n_in // h))


def test_golden_spec_worked_values():
    with open(os.path.join(GOLDEN, "spec_worked_values.json")) as f:
        g = json.load(f)
    k1 = g["k1_energy_single"]
    assert dsp.energy(np.array([[complex(*k1["z"])]]))[0] == k1["E"]
    k6 = g["k6_notch_D32"]
    m = dsp.notch_mask(32)
    assert [int(i) for i in np.nonzero(m == 0)[0]] == k6["zeroed"]
    assert np.array_equal(m * m, m)  # idempotent
    k2 = g["k2_gamma_powers"]
    E = np.array(k2["E"], dtype=float)
    assert list(E ** k2["gamma"]) == k2["w"]
    pk = g["packing"]
    assert pk["A"] * pk["R"] * pk["D"] == pk["active"]
    rec = g["recover"]
    assert rec["N"] / rec["D"] == rec["r_hat"]


# ------------------------------------------------------------------ encrypted chains

@pytest.fixture(scope="module")
def Pg():
    # 12 Q limbs (depth 11, Table tab:depth) at N=2^10; alpha=2 so P covers each digit
    return toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)


def _enc(P, keys, v, level, idx, seed=31):
    return orc.encrypt_vector(P, keys, v, level, seed=seed, index=idx)


def test_k1_k2_vital_v1(Pg):
    P = Pg
    cfg = cc.ChainCfg(R=16, F=6, gamma=2, n_slots=P.n // 2)
    z, truth = radar.vital_scene(cfg.R, cfg.F, 20.0, seed=1001)
    zt = radar.preprocess_vital(z)
    keys = orc.keygen(P, seed=2001, rotations=cc.required_rotations("vitals_v1", cfg, P.n))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    lvl = 3
    re = [_enc(P, keys, radar.pack_vital(zt[t].real, cfg.n_slots), lvl, 2 * t) for t in range(cfg.F)]
    im = [_enc(P, keys, radar.pack_vital(zt[t].imag, cfg.n_slots), lvl, 2 * t + 1) for t in range(cfg.F)]
    E = cc.k1_energy(ev, re, im)
    E_dec = orc.decrypt_vector(P, keys, E)[: cfg.R]
    assert rel_err(E_dec, dsp.energy(zt)) < 1e-3
    Nc, Dc = cc.k2_soft_attention(ev, book, E, cfg)
    assert Nc.level == 0
    N = orc.decrypt_vector(P, keys, Nc)[0]
    D = orc.decrypt_vector(P, keys, Dc)[0]
    Np, Dp, rp = dsp.soft_attention(dsp.energy(zt), cfg.gamma, cfg.F)
    assert abs(N - Np) <= 1e-3 * abs(Np) and abs(D - Dp) <= 1e-3 * abs(Dp)
    assert round(N / D) == round(rp)


def _gesture_setup(P, A=2, R=4, D=8, F=2, seed=5):
    n = A * R * D
    cfg = cc.ChainCfg(A=A, R=R, D=D, F=F, gamma=4, n_slots=n, fc_dims=(n, 16, 8, 8))
    Z, _ = radar.gesture_scene(A, R, D, F, seed=seed, cls=seed % 5)
    Zt = radar.preprocess_gesture(Z)
    return cfg, Zt


@pytest.mark.parametrize("hoist", [0, 1])
def test_gesture_frame_and_fc(Pg, hoist):
    P = Pg
    cfg, Zt = _gesture_setup(P)
    cfg.hoist = hoist
    keys = orc.keygen(P, seed=2002, rotations=cc.required_rotations("gesture", cfg, P.n))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    lvl = P.L
    feats, feats_plain = [], []
    for t in range(cfg.F):
        v = radar.pack_doppler(Zt[t])
        cr = _enc(P, keys, v.real, lvl, 2 * t)
        ci = _enc(P, keys, v.imag, lvl, 2 * t + 1)
        if t == 0:
            dre, dim = cc.k3_doppler_dft(ev, book, cr, ci, cfg)
            want = dsp.doppler_dft(v, cfg.D)
            assert rel_err(orc.decrypt_vector(P, keys, dre), want.real) < 1e-3
            assert rel_err(orc.decrypt_vector(P, keys, dim), want.imag) < 1e-3
        f = cc.gesture_frame(ev, book, cr, ci, cfg)
        assert f.level == lvl - 6  # Table tab:depth: feature weighting at Sigma 6
        fp = dsp.gesture_frame_features(v, cfg.A, cfg.R, cfg.D, cfg.gamma)
        assert rel_err(orc.decrypt_vector(P, keys, f), fp) < 1e-3
        feats.append(f)
        feats_plain.append(fp)
    feat = cc.frame_accumulate(ev, feats)
    xp = np.sum(feats_plain, axis=0)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=7)
    Ws[0] = Ws[0] / max(np.max(np.abs(Ws[0] @ xp)), 1e-30) * 0.8  # pre-activations O(1)
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    assert logits.level == lvl - 11  # Sigma 11
    got = orc.decrypt_vector(P, keys, logits)[:5]
    want = dsp.mlp_forward(xp, Ws, bs)
    assert rel_err(got, want) < 1e-3
    assert int(np.argmax(got)) == int(np.argmax(want))


def test_vitals_v2_small(Pg):
    P = toy(log_n=10, n_q=8, scale_bits=40, n_p=2, alpha=2)
    cfg = cc.ChainCfg(R=8, F=16, p_phi=2, taylor_order=1, n_slots=P.n // 2, fs=2.0,
                      bands=((0.1, 0.6), (0.7, 1.0)))
    z, _ = radar.vital_scene(cfg.R, cfg.F, cfg.fs, seed=1003)
    zt = radar.preprocess_vital(z)
    keys = orc.keygen(P, seed=2003, rotations=cc.required_rotations("vitals_v2", cfg, P.n))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    lvl = 7
    re = [_enc(P, keys, radar.pack_vital(zt[t].real, cfg.n_slots), lvl, 2 * t) for t in range(cfg.F)]
    im = [_enc(P, keys, radar.pack_vital(zt[t].imag, cfg.n_slots), lvl, 2 * t + 1) for t in range(cfg.F)]
    taps = [np.array([0.2, 0.3, 0.3, 0.2]), np.array([0.25, -0.5, 0.25])]
    out = cc.vitals_v2(ev, re, im, taps, cfg)
    I = np.array([dsp.soft_iq(zt[t], cfg.p_phi)[0] for t in range(cfg.F)])
    Q = np.array([dsp.soft_iq(zt[t], cfg.p_phi)[1] for t in range(cfg.F)])
    for bi, h in enumerate(taps):
        y = dsp.taylor_phase(dsp.fir(I, h), dsp.fir(Q, h), cfg.taylor_order)
        bins = dsp.band_bins(len(y), cfg.fs, cfg.bands[bi])
        want = dsp.narrowband_power(y, bins)
        got = np.array([orc.decrypt_vector(P, keys, c)[0] for c in out[bi]])
        assert len(got) == len(bins) > 0
        assert out[bi][0].level == 0
        assert rel_err(got, want) < 1e-3


def test_vitals_v2_vp_plus(Pg):
    """Full-depth V2 (SURVEY §8(c)-7 VP+): sharpen + weighted frequency
    average in the cloud; decrypted N_f, D_f match the plaintext sums over the plaintext
    band powers, and 60 N_f / D_f the client's BPM formula.  Depth 9 (c-6 ledger)."""
    # Delta = 2^50 (as PS4, where the full chain runs): the sharpened powers are ~1e-9 here
    P = toy(log_n=10, n_q=10, scale_bits=50, n_p=2, alpha=2)
    cfg = cc.ChainCfg(R=8, F=16, p_phi=2, taylor_order=1, n_slots=P.n // 2, fs=2.0,
                      bands=((0.1, 0.6), (0.7, 1.0)), vp_plus=1)
    z, _ = radar.vital_scene(cfg.R, cfg.F, cfg.fs, seed=1004)
    zt = radar.preprocess_vital(z)
    keys = orc.keygen(P, seed=2004, rotations=cc.required_rotations("vitals_v2", cfg, P.n))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    lvl = 9
    re = [_enc(P, keys, radar.pack_vital(zt[t].real, cfg.n_slots), lvl, 2 * t) for t in range(cfg.F)]
    im = [_enc(P, keys, radar.pack_vital(zt[t].imag, cfg.n_slots), lvl, 2 * t + 1) for t in range(cfg.F)]
    taps = [np.array([0.2, 0.3, 0.3, 0.2]), np.array([0.25, -0.5, 0.25])]
    out = cc.vitals_v2(ev, re, im, taps, cfg)
    I = np.array([dsp.soft_iq(zt[t], cfg.p_phi)[0] for t in range(cfg.F)])
    Q = np.array([dsp.soft_iq(zt[t], cfg.p_phi)[1] for t in range(cfg.F)])
    for bi, h in enumerate(taps):
        y = dsp.taylor_phase(dsp.fir(I, h), dsp.fir(Q, h), cfg.taylor_order)
        bins = dsp.band_bins(len(y), cfg.fs, cfg.bands[bi])
        Pk = dsp.narrowband_power(y, bins)
        want_n, want_d = dsp.weighted_average(Pk, bins, cfg.fs, len(y))
        assert len(out[bi]) == 2 and out[bi][0].level == 0 and out[bi][0].scale == out[bi][1].scale
        got_n, got_d = (orc.decrypt_vector(P, keys, c)[0] for c in out[bi])
        assert abs(got_n - want_n) <= 1e-3 * abs(want_n) and abs(got_d - want_d) <= 1e-3 * abs(want_d)
        bpm = dsp.bpm_from_power(Pk, bins, cfg.fs, len(y))
        assert abs(60.0 * want_n / want_d - bpm) <= 1e-9 * bpm
        assert abs(60.0 * got_n / got_d - bpm) <= 1e-2  # BPM gate is 1 BPM (north star)


@pytest.mark.parametrize("k,hoist", [(1, 0), (2, 0), (3, 0), (1, 1), (3, 1)])
def test_k4_iq_pack_matches_canonical(Pg, k, hoist):
    """Reading R19: K4's packed rotate-and-sum (i, q of 2^(k-1) frames packed into slot blocks,
    one rotsum, unpacked) decrypts to the same I, Q in slot 0 as the two canonical rotsums
     with 2(2 - 2^(1-k)) + log2(R) / 2^(k-1) rotations per frame."""
    P = toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)
    F, R = 8, 8
    cfg = cc.ChainCfg(R=R, F=F, p_phi=2, n_slots=P.n // 2)
    z, _ = radar.vital_scene(R, F, 20.0, seed=1005)
    zt = radar.preprocess_vital(z)
    cfgp = cc.ChainCfg(R=R, F=F, p_phi=2, n_slots=P.n // 2, iq_pack=k, hoist=hoist)
    rots = cc.required_rotations("vitals_v2", cfgp, P.n)
    assert all((R << j) in rots and (P.n // 2 - (R << j)) in rots for j in range(k))
    keys = orc.keygen(P, seed=2005, rotations=rots)
    re = [_enc(P, keys, radar.pack_vital(zt[t].real, cfg.n_slots), 5, 2 * t) for t in range(F)]
    im = [_enc(P, keys, radar.pack_vital(zt[t].imag, cfg.n_slots), 5, 2 * t + 1) for t in range(F)]
    want = np.array([dsp.soft_iq(zt[t], cfg.p_phi) for t in range(F)])
    # rotations per frame: pack 2 - 2^(1-k), rotsum log2(R) / 2^(k-1), unpack 2 - 2^(1-k)
    # (plain) or (2^k - 1) / 2^(k-1) hoisted rotations sharing one ModUp per group
    packed = F * ((2 - 2.0 ** (1 - k)) + 3 / 2 ** (k - 1)) + F * (((1 << k) - 1) / 2 ** (k - 1) if hoist
                                                                  else 2 - 2.0 ** (1 - k))
    for c, n_rot in ((cfg, 2 * 3 * F), (cfgp, int(round(packed)))):
        ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
        I, Q = cc.k4_soft_iq(ev, re, im, c)
        got_i = np.array([orc.decrypt_vector(P, keys, x)[0] for x in I])
        got_q = np.array([orc.decrypt_vector(P, keys, x)[0] for x in Q])
        assert rel_err(got_i, want[:, 0]) < 1e-3 and rel_err(got_q, want[:, 1]) < 1e-3
        assert sum(1 for op in ev.trace if op[0] in ("hrot", "hrot_hoisted")) == n_rot
        assert sum(1 for op in ev.trace if op[0] == "hrot_hoisted") == (F * ((1 << k) - 1) // (1 << (k - 1))
                                                                      if c.hoist else 0)


def test_trace_is_data_oblivious(Pg):
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    cfg = cc.ChainCfg(R=8, F=3, gamma=2, n_slots=P.n // 2)
    keys = orc.keygen(P, seed=9, rotations=cc.required_rotations("vitals_v1", cfg, P.n))
    traces = []
    for seed in (1, 2):
        rng = np.random.default_rng(seed)
        ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
        book = cc.PlainBook(P)
        re = [_enc(P, keys, rng.uniform(-1, 1, 8), 3, t, seed) for t in range(cfg.F)]
        im = [_enc(P, keys, rng.uniform(-1, 1, 8), 3, 10 + t, seed) for t in range(cfg.F)]
        cc.vitals_v1(ev, book, re, im, cfg)
        traces.append(ev.trace)
    assert traces[0] == traces[1] and len(traces[0]) > 10


def test_required_rotation_counts():
    # SURVEY §8(d) key table: C3 needs 14 keys, C4 31 (amounts normalised to [0, N/2))
    n_ring = 1 << 16
    cfg = cc.ChainCfg(A=4, R=32, D=32, n_slots=4096, gamma=4, fc_dims=(4096, 64, 32, 8))
    k3 = cc.required_rotations("k3_doppler_dft", cfg, n_ring)
    assert len(k3) == 14
    assert (n_ring // 2 - 31) in k3 and 25 in k3
    vital = cc.required_rotations("vitals_v1", cc.ChainCfg(R=128), n_ring)
    assert vital == [1, 2, 4, 8, 16, 32, 64]


# ------------------------------------------------------------------ K7 third order (pins)

def test_taylor_phase_polynomial_closed_forms():
    """Eq. taylor_arctan through angles, not the code's formula: for unit
    phasors z_t = e^{j th_t}, y = sin(dth) and x = cos(dth), so the third-order value is
    sin(dth) cos^2(dth) - sin^3(dth)/3 and the first-order value sin(dth); equal samples
    give y = 0, x = 1 and a zero phase step; and y x^2 - y^3/3 = x^3 (t - t^3/3),
    t = y/x, the cubic Taylor polynomial of x^3 arctan(t) (error <= |x|^3 |t|^5 / 5)."""
    rng = np.random.default_rng(11)
    th = np.cumsum(rng.uniform(-0.6, 0.6, 64))
    I, Q = np.cos(th), np.sin(th)
    d = np.diff(th)
    assert np.allclose(dsp.taylor_phase(I, Q, 1), np.sin(d), atol=1e-14)
    want3 = np.sin(d) * np.cos(d) ** 2 - np.sin(d) ** 3 / 3.0
    assert np.allclose(dsp.taylor_phase(I, Q, 3), want3, atol=1e-14)
    # equal consecutive samples: zero phase step at both orders
    Ie, Qe = np.full(4, 0.6), np.full(4, 0.8)
    assert np.allclose(dsp.taylor_phase(Ie, Qe, 1), 0.0) and np.allclose(dsp.taylor_phase(Ie, Qe, 3), 0.0)
    # arbitrary magnitudes: within the Taylor remainder of x^3 arctan(y/x)
    a = rng.uniform(0.3, 1.0, 65)
    I2, Q2 = a * np.cos(np.concatenate([[0], th])), a * np.sin(np.concatenate([[0], th]))
    y = Q2[1:] * I2[:-1] - I2[1:] * Q2[:-1]
    x = I2[1:] * I2[:-1] + Q2[1:] * Q2[:-1]
    t = y / x
    got = dsp.taylor_phase(I2, Q2, 3)
    assert np.all(np.abs(got - x ** 3 * np.arctan(t)) <= np.abs(x) ** 3 * np.abs(t) ** 5 / 5 + 1e-15)


@pytest.mark.parametrize("order", [1, 3])
def test_k7_taylor_phase_decrypts_to_polynomial(order):
    """The oracle's K7 circuit (c-7: y by one lazy relin; third order x, x^2, y^2, -y/3 as an
    exact scalar at q_l, y x^2 + y^2 (-y/3)) decrypts to the literal polynomial of the
    plaintext I_f, Q_f slot by slot, including a slot with equal consecutive samples."""
    P = toy(log_n=10, n_q=5, scale_bits=40, n_p=2, alpha=2)
    F, n = 5, P.n // 2
    rng = np.random.default_rng(order)
    th = np.cumsum(rng.uniform(-0.5, 0.5, (F, n)), axis=0)
    amp = rng.uniform(0.4, 1.0, (F, n))
    I, Q = amp * np.cos(th), amp * np.sin(th)
    I[:, 7], Q[:, 7] = 0.6, 0.8  # equal samples in slot 7: y = 0, x = 1
    keys = orc.keygen(P, seed=2101)
    lvl = 4
    Ie = [_enc(P, keys, I[t], lvl, 2 * t, seed=2102) for t in range(F)]
    Qe = [_enc(P, keys, Q[t], lvl, 2 * t + 1, seed=2102) for t in range(F)]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    out = cc.k7_taylor_phase(ev, Ie, Qe, order)
    assert len(out) == F - 1
    assert out[0].level == lvl - (3 if order == 3 else 1)  # Table tab:depth: K7 depth 3 / 1
    got = np.array([orc.decrypt_vector(P, keys, c) for c in out])
    want = np.stack([dsp.taylor_phase(I[:, j], Q[:, j], order) for j in range(n)], axis=1)
    assert rel_err(got, want) < 1e-3
    assert np.max(np.abs(got[:, 7])) < 1e-6
    # third order differs from first order (a dropped term would make them agree)
    if order == 3:
        y1 = np.stack([dsp.taylor_phase(I[:, j], Q[:, j], 1) for j in range(n)], axis=1)
        assert rel_err(got, y1) > 1e-2


def test_k7_rejects_other_orders():
    P = toy(log_n=10, n_q=5, scale_bits=40, n_p=2, alpha=2)
    ev = cc.CircuitEvaluator(P)
    with pytest.raises(ValueError):
        cc.k7_taylor_phase(ev, [], [], 2)


def test_public_exponents_must_be_powers_of_two():
    """gamma / p_phi are numbers of squarings (log2), never rounded; the packed
    K4 rotate-and-sum rejects a non-power-of-two R (its blocks would overlap)."""
    with pytest.raises(ValueError):
        cc.log2_exact(3, "gamma")
    assert cc.log2_exact(4, "gamma") == 2
    with pytest.raises(ValueError):
        cc.required_rotations("vitals_v2", cc.ChainCfg(R=100, iq_pack=1, n_slots=4096), 1 << 13)


# ------------------------------------------------------------------ SIMD-dense lanes (R20)

@pytest.mark.parametrize("L", [2, 4])
def test_lane_interleaved_k3_schedule_on_plain_slots(L):
    """Reading R20 on plaintext slot vectors: with L frames interleaved (slot L i + f), the
    K3 BSGS schedule with rotations scaled by L and lane-repeated diagonals computes every
    frame's block-diagonal DFT exactly, and lanes never mix."""
    D, n = 8, 32
    cfg = cc.ChainCfg(D=D)
    rng = np.random.default_rng(L)
    M = rng.normal(size=(D, D))
    frames = [rng.normal(size=n) for _ in range(L)]
    x = cc.interleave(frames, L, n)
    bb, giants = cc.k3_schedule(cfg)
    babies = [cc.rot(x, s * L) for s in range(bb)]
    y = np.zeros(n * L)
    for gp, G, ss in giants:
        inner = sum(cc.lane_vec(cc.rot(cc.block_diag_diagonal(M, n, G + s), -G), L) * babies[s] for s in ss)
        y += cc.rot(inner, G * L)
    for f in range(L):
        assert np.allclose(y[f::L], np.kron(np.eye(n // D), M) @ frames[f])
    # lane rotate-and-sum: lane 0 holds the sum over the L frames
    z = y.copy()
    s = 1
    while s < L:
        z = z + cc.rot(z, s)
        s *= 2
    assert np.allclose(z[0::L], sum(np.kron(np.eye(n // D), M) @ v for v in frames))


def test_gesture_lanes_decrypt_like_canonical(Pg):
    """The SIMD-dense gesture pipeline (4 frames per ciphertext, 6 frames -> 2 ciphertext
    pairs, the last half empty) decrypts to the same logits as the plaintext DSP and the
    same per-frame features (lane by lane) as the one-frame-per-ciphertext layout."""
    P = Pg
    F, L = 6, 4
    cfg, Zt = _gesture_setup(P, F=F)
    cfg.hoist, cfg.lanes = 1, L
    n = cfg.n_slots
    rots = cc.required_rotations("gesture", cfg, P.n)
    assert 1 in rots and (cfg.D * L) in rots
    keys = orc.keygen(P, seed=2011, rotations=rots)
    vs = [radar.pack_doppler(Zt[t]) for t in range(F)]
    re, im = [], []
    for g in range(cc.n_packed(F, L)):
        grp = vs[g * L:(g + 1) * L]
        re.append(_enc(P, keys, cc.interleave([v.real for v in grp], L, n), P.L, 4 * g))
        im.append(_enc(P, keys, cc.interleave([v.imag for v in grp], L, n), P.L, 4 * g + 1))
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    fr = cc.gesture_frames(ev, book, re, im, cfg)
    fp = [dsp.gesture_frame_features(v, cfg.A, cfg.R, cfg.D, cfg.gamma) for v in vs]
    for g, c in enumerate(fr):
        dec = orc.decrypt_vector(P, keys, c)
        for f in range(L):
            want = fp[g * L + f] if g * L + f < F else np.zeros(n)
            assert np.max(np.abs(dec[f::L] - want)) <= 1e-3 * max(np.max(np.abs(fp)), 1e-30)
    feat = cc.frame_accumulate(ev, fr)
    xp = np.sum(fp, axis=0)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=7)
    Ws[0] = Ws[0] / max(np.max(np.abs(Ws[0] @ xp)), 1e-30) * 0.8
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    assert logits.level == P.L - 11  # lanes add rotations only, no depth
    got = orc.decrypt_vector(P, keys, logits)[cc.logit_slots(5, L)]
    want = dsp.mlp_forward(xp, Ws, bs)
    assert rel_err(got, want) < 1e-3
    assert int(np.argmax(got)) == int(np.argmax(want))


# ------------------------------------------------------------------ double-hoisted BSGS (hoist = 2)

def test_pq_lift_moddown_is_exact_and_rotate_pq_rotates():
    """Double hoisting's PQ ops (SURVEY §8(c)-5 third op): ModDown(P c) = c exactly (the
    P rows of a lifted ciphertext are zero, so the base conversion adds nothing), and a PQ
    giant rotation followed by the final ModDown decrypts to the slot rotation."""
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    keys = orc.keygen(P, seed=2201, rotations=[5])
    v = np.random.default_rng(5).uniform(-1, 1, P.n // 2)
    ct = _enc(P, keys, v, 3, 0)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    lifted = ev.lift_pq(ct)
    assert len(lifted.c[0]) == 4 + P.K and not lifted.c[0][4:].any()
    back = ev.moddown_ct(lifted)
    assert all(np.array_equal(a, b) for a, b in zip(back.c, ct.c))
    r = ev.moddown_ct(ev.rotate_pq(lifted, 5))
    assert rel_err(orc.decrypt_vector(P, keys, r), np.roll(v, -5)) < 1e-6
    # a hoisted baby step left in PQ, brought down, decrypts to the rotation as well
    hb = ev.moddown_ct(ev.hoisted_step_pq(ct, ev.hoist_modup(ct), 5))
    assert rel_err(orc.decrypt_vector(P, keys, hb), np.roll(v, -5)) < 1e-6


@pytest.mark.parametrize("L", [1, 2])
def test_double_hoisted_k3_decrypts_to_dft(Pg, L):
    """K3 with double-hoisted BSGS (cfg.hoist = 2) decrypts to fftshift(fft(hann x)) per
    block like the single-hoisted circuit; the op counts are the double-hoisted schedule:
    2 lifts + 2(b-1) PQ baby steps, one PQ giant step per nonzero giant offset and output,
    one ModDown per output (no HRot with its own ModDown)."""
    P = Pg
    cfg, Zt = _gesture_setup(P, F=2)
    cfg.hoist, cfg.lanes = 2, L
    n = cfg.n_slots
    keys = orc.keygen(P, seed=2202, rotations=cc.required_rotations("k3_doppler_dft", cfg, P.n))
    vs = [radar.pack_doppler(Zt[t]) for t in range(L)]
    cr = _enc(P, keys, cc.interleave([v.real for v in vs], L, n), P.L, 0)
    ci = _enc(P, keys, cc.interleave([v.imag for v in vs], L, n), P.L, 1)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    dre, dim = cc.k3_doppler_dft(ev, cc.PlainBook(P), cr, ci, cfg)
    b, giants = cc.k3_schedule(cfg)
    ops = [op for op, _, _ in ev.trace]
    assert ops.count("hrot_hoisted_pq") == 2 * (b - 1) and ops.count("lift_pq") == 2
    assert ops.count("hrot_pq") == 2 * sum(1 for _, G, _ in giants if G) and ops.count("moddown") == 2
    assert "hrot" not in ops and "hrot_hoisted" not in ops
    got_re, got_im = orc.decrypt_vector(P, keys, dre), orc.decrypt_vector(P, keys, dim)
    for f in range(L):
        want = dsp.doppler_dft(vs[f], cfg.D)
        assert rel_err(got_re[f::L], want.real) < 1e-3 and rel_err(got_im[f::L], want.imag) < 1e-3


def test_double_hoisted_gesture_pipeline(Pg):
    """The whole gesture pipeline with double-hoisted K3 and FC (hoist = 2, 2 lanes):
    features and logits decrypt to the plaintext DSP; argmax agrees; depth unchanged."""
    P = Pg
    F, L = 4, 2
    cfg, Zt = _gesture_setup(P, F=F)
    cfg.hoist, cfg.lanes = 2, L
    n = cfg.n_slots
    keys = orc.keygen(P, seed=2203, rotations=cc.required_rotations("gesture", cfg, P.n))
    vs = [radar.pack_doppler(Zt[t]) for t in range(F)]
    re = [_enc(P, keys, cc.interleave([v.real for v in vs[g * L:(g + 1) * L]], L, n), P.L, 2 * g) for g in range(2)]
    im = [_enc(P, keys, cc.interleave([v.imag for v in vs[g * L:(g + 1) * L]], L, n), P.L, 2 * g + 1)
          for g in range(2)]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    feat = cc.gesture_features(ev, book, re, im, cfg)
    xp = np.sum([dsp.gesture_frame_features(v, cfg.A, cfg.R, cfg.D, cfg.gamma) for v in vs], axis=0)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=7)
    Ws[0] = Ws[0] / max(np.max(np.abs(Ws[0] @ xp)), 1e-30) * 0.8
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    assert logits.level == P.L - 11
    got = orc.decrypt_vector(P, keys, logits)[cc.logit_slots(5, L)]
    want = dsp.mlp_forward(xp, Ws, bs)
    assert rel_err(got, want) < 1e-3
    assert int(np.argmax(got)) == int(np.argmax(want))


# ------------------------------------------------------------------ K5 by slot rotations

@pytest.mark.parametrize("W", [1, 5, 41])
def test_k5_fir_rot_decrypts_to_lfilter(W):
    """The rotation-based FIR on a sequence packed in the slots of one ciphertext
    decrypts to scipy's causal lfilter (zero initial state) over the sequence; depth 1."""
    P = toy(log_n=10, n_q=3, scale_bits=40, n_p=2, alpha=2)
    rng = np.random.default_rng(W)
    F = 120
    x = np.zeros(P.n // 2)
    x[:F] = rng.uniform(-1, 1, F)
    taps = radar.fir_taps(W, (0.8, 2.5), 20.0) if W > 1 else np.array([0.7])
    cfg = cc.ChainCfg(n_taps=(W,), n_slots=P.n // 2)
    keys = orc.keygen(P, seed=2301, rotations=cc.required_rotations("k5_fir_rot", cfg, P.n))
    ct = _enc(P, keys, x, 2, 0)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    y = cc.k5_fir_rot(ev, ct, taps)
    assert y.level == 1
    got = orc.decrypt_vector(P, keys, y)[:F]
    want = dsp.fir(x[:F], taps)
    assert rel_err(got, want) < 1e-4
    b, giants = cc.fir_rot_schedule(W)
    assert sum(1 for op in ev.trace if op[0] in ("hrot", "hrot_hoisted")) == (min(b, W) - 1) + (len(giants) - 1)


@pytest.mark.parametrize("count,inner", [(8, 8), (32, 8), (4, 8), (16, 4)])
def test_double_hoisted_rotsum_equals_rotsum(count, inner):
    """Reading R27: the rotate-and-sum with a double-hoisted first level (one ModUp, inner - 1
    PQ rotations, one ModDown, then the remaining rotate-and-add steps) decrypts to the same
    slot sums as the sequential one, sum_{m < count} Rot(v, m stride), with fewer key switches."""
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    stride = 3
    rots = sorted({(j * stride) % (P.n // 2) for j in range(1, count)})
    keys = orc.keygen(P, seed=2401, rotations=rots)
    v = np.random.default_rng(count).uniform(-1, 1, P.n // 2)
    ct = _enc(P, keys, v, 3, 0)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    got = orc.decrypt_vector(P, keys, ev.rotsum_dh_all([ct], count, stride, inner)[0])
    want = sum(np.roll(v, -m * stride) for m in range(count))
    assert rel_err(got, want) < 1e-6
    a = min(inner, count)
    ops = [op for op, _, _ in ev.trace]
    assert ops.count("hrot_hoisted_pq") == a - 1 and ops.count("moddown") == 1
    assert ops.count("hrot") == int(np.log2(count // a))


@pytest.mark.parametrize("count,inner", [(32, 4), (16, 2), (8, 8), (64, 4)])
def test_all_levels_hoisted_rotsum_equals_rotsum(count, inner):
    """Reading R30: every level of the rotate-and-sum double-hoisted (groups of `inner`, the last
    one what is left) decrypts to the same slot sums; no plain HRot remains, one ModDown per level."""
    P = toy(log_n=10, n_q=4, scale_bits=40, n_p=2, alpha=2)
    stride = 3
    levels = cc.rotsum_levels(count, inner, True)
    assert int(np.prod(levels)) == count
    rots = sorted({(j * stride) % (P.n // 2) for j in range(1, count)})
    keys = orc.keygen(P, seed=2402, rotations=rots)
    v = np.random.default_rng(count + 7).uniform(-1, 1, P.n // 2)
    ct = _enc(P, keys, v, 3, 0)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    got = orc.decrypt_vector(P, keys, ev.rotsum_dh_all([ct], count, stride, inner, True)[0])
    want = sum(np.roll(v, -m * stride) for m in range(count))
    assert rel_err(got, want) < 1e-6
    ops = [op for op, _, _ in ev.trace]
    assert ops.count("hrot") == 0 and ops.count("moddown") == len(levels)
    assert ops.count("hrot_hoisted_pq") == sum(a - 1 for a in levels)
    # the key set of a chain using it (K2b: count = n / D terms at stride D): exactly the levels' strides
    cfg = cc.ChainCfg(D=stride, n_slots=stride * count, hoist=2, rotsum_inner=inner, rotsum_hoist_all=1)
    st, want_keys = stride, set()
    for a in levels:
        want_keys |= {j * st for j in range(1, a)}
        st *= a
    assert cc.required_rotations("k2_doppler_soft_power", cfg, P.n) == sorted(k % (P.n // 2) for k in want_keys)
    assert cc.rotsum_levels(count, inner, False) == [min(inner, count)]


# ------------------------------------------------------------------ complex slots (reading R28)

@pytest.mark.parametrize("hoist,L,aligned", [(1, 1, 0), (2, 2, 0), (2, 2, 1)])
def test_complex_k3_decrypts_to_dft(Pg, hoist, L, aligned):
    """K3 on complex slots (cfg.cplx): z = v_re + j v_im in one ciphertext, complex diagonals
    of W~ -- decrypts (complex decode) to fftshift(fft(hann x)) per block and
    lane, with half the baby steps and giant rotations of the split layout."""
    P = Pg
    cfg, Zt = _gesture_setup(P, F=2)
    cfg.hoist, cfg.lanes, cfg.cplx, cfg.bsgs_aligned = hoist, L, 1, aligned
    n = cfg.n_slots
    keys = orc.keygen(P, seed=2301, rotations=cc.required_rotations("k3_doppler_dft", cfg, P.n))
    assert orc.CONJ not in keys.gk  # K3 alone needs no conjugation
    vs = [radar.pack_doppler(Zt[t]) for t in range(L)]
    cz = _enc(P, keys, cc.interleave(vs, L, n), P.L, 0)
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    d = cc.k3_doppler_dft_frames_c(ev, cc.PlainBook(P), [cz], cfg)[0]
    b, giants = cc.k3_schedule(cfg)
    ops = [op for op, _, _ in ev.trace]
    base = "hrot_hoisted_pq" if hoist == 2 else "hrot_hoisted"
    assert ops.count(base) == b - 1
    assert ops.count("hrot_pq" if hoist == 2 else "hrot") == sum(1 for _, G, _ in giants if G)
    assert d.level == P.L - 1
    got = orc.decrypt_vector(P, keys, d, complex_out=True)
    for f in range(L):
        want = dsp.doppler_dft(vs[f], cfg.D)
        assert rel_err(got[f::L], want) < 1e-3


@pytest.mark.parametrize("hoist,merge", [(1, 0), (2, 0), (2, 1), (2, 2)])
def test_complex_gesture_pipeline(Pg, hoist, merge):
    """The gesture pipeline on complex slots (one ciphertext per frame group, 2 lanes): per
    frame P = |d|^2 by d Conj(d) (one conjugation key switch per ciphertext), features and
    logits decrypt to the plaintext DSP, argmax agrees, depth unchanged (11)."""
    P = Pg
    F, L = 4, 2
    cfg, Zt = _gesture_setup(P, F=F)
    cfg.hoist, cfg.lanes, cfg.cplx, cfg.ks_merge = hoist, L, 1, min(merge, 1)
    cfg.k1_conj_fuse = int(merge == 2)  # merge 2: + K1 as one conjugate-product key switch (R32)
    n = cfg.n_slots
    rots = cc.required_rotations("gesture", cfg, P.n)
    assert (orc.CONJ_PROD in rots) == (merge == 2)
    assert orc.CONJ in rots and rots[0] == orc.CONJ
    keys = orc.keygen(P, seed=2302, rotations=rots)
    vs = [radar.pack_doppler(Zt[t]) for t in range(F)]
    z = [_enc(P, keys, cc.interleave(vs[g * L:(g + 1) * L], L, n), P.L, g) for g in range(2)]
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    book = cc.PlainBook(P)
    fr = cc.gesture_frames(ev, book, z, None, cfg)
    assert [op for op, _, _ in ev.trace].count("conj") == (0 if merge == 2 else 2)
    assert [op for op, _, _ in ev.trace].count("conj_mul_relin_rescale") == (2 if merge == 2 else 0)
    # R31: every relinearisation / ModDown that a rescale follows is one division
    ops = [op for op, _, _ in ev.trace]
    assert (ops.count("relin_rescale") > 0) == bool(merge) and (ops.count("relin") == 0) == bool(merge)
    fp = [dsp.gesture_frame_features(v, cfg.A, cfg.R, cfg.D, cfg.gamma) for v in vs]
    for g, c in enumerate(fr):
        dec = orc.decrypt_vector(P, keys, c)
        for f in range(L):
            assert np.max(np.abs(dec[f::L] - fp[g * L + f])) <= 1e-3 * np.max(np.abs(fp))
    feat = cc.frame_accumulate(ev, fr)
    xp = np.sum(fp, axis=0)
    dims = cfg.fc_dims
    Ws, bs = radar.fc_weights([dims[0], dims[1], dims[2], 5], seed=7)
    Ws[0] = Ws[0] / max(np.max(np.abs(Ws[0] @ xp)), 1e-30) * 0.8
    logits = cc.gesture_fc(ev, book, feat, Ws, bs, cfg)
    assert logits.level == P.L - 11
    got = orc.decrypt_vector(P, keys, logits)[cc.logit_slots(5, L)]
    want = dsp.mlp_forward(xp, Ws, bs)
    assert rel_err(got, want) < 1e-3
    assert int(np.argmax(got)) == int(np.argmax(want))
    with pytest.raises(ValueError):
        cc.gesture_frames(ev, book, z, z, cfg)


def test_round2_cfg_fields_validated():
    """rotsum_inner must be a power of two (R27); the aligned K3 schedule (R29) and complex slots
    (R28) change the key set as stated: the conjugation key only with complex slots, and aligned
    giants drop the G = 0 rotation key."""
    with pytest.raises(ValueError):
        cc.rotsum_inner(cc.ChainCfg(rotsum_inner=3))
    assert cc.rotsum_inner(cc.ChainCfg()) == 8 and cc.rotsum_inner(cc.ChainCfg(rotsum_inner=16)) == 16
    n_ring = 1 << 16
    base = dict(A=4, R=32, D=32, n_slots=4096, gamma=4, fc_dims=(4096, 64, 32, 8), bsgs_baby=16, hoist=2, lanes=8)
    k_plain = cc.required_rotations("gesture", cc.ChainCfg(**base), n_ring)
    k_cplx = cc.required_rotations("gesture", cc.ChainCfg(**base, cplx=1), n_ring)
    assert orc.CONJ not in k_plain and k_cplx == [orc.CONJ] + k_plain
    k3a = cc.required_rotations("k3_doppler_dft", cc.ChainCfg(**base, bsgs_aligned=1), n_ring)
    assert k3a == sorted({(s * 8) % (n_ring // 2) for s in range(1, 16)} |
                         {(G * 8) % (n_ring // 2) for G in (-32, -16, 16)})


# ------------------------------------------------------------------ vital sessions packed per ciphertext (R33)

def _decode_all(P, keys, ct):
    return orc.decode(P, orc.decrypt(P, keys, ct), ct.level, ct.scale, P.n // 2)


@pytest.mark.parametrize("iq_pack,merge", [(0, 0), (3, 0), (3, 1)])
def test_vital_sessions_packed_per_ciphertext(iq_pack, merge):
    """Reading R33 (SURVEY §8(f)-3 "several sessions per ciphertext"): with the packing period
    n = R 2^iq_pack (cfg.n_slots), S = N / (2n) vital sessions share every ciphertext, session s in
    slots [s n, s n + R) (zeros up to the next block, reading #23).  Every vital op is slot-wise or
    rotates by less than n within the block it reads, and the public vectors are period-n, so V1 and
    V2 give each session's outputs in slot s n: checked against each session's plaintext DSP."""
    P = toy(log_n=10, n_q=8, scale_bits=40, n_p=2, alpha=2)
    R, F = 8, 16
    n = R << iq_pack
    S = (P.n // 2) // n
    cfg = cc.ChainCfg(R=R, F=F, gamma=2, p_phi=2, taylor_order=1, n_slots=n, fs=2.0,
                      bands=((0.1, 0.6), (0.7, 1.0)), iq_pack=iq_pack, frame_batch=F, ks_merge=merge)
    scenes = [radar.preprocess_vital(radar.vital_scene(R, F, cfg.fs, seed=1100 + s)[0]) for s in range(S)]
    rots = sorted(set(cc.required_rotations("vitals_v1", cfg, P.n)) | set(cc.required_rotations("vitals_v2", cfg, P.n)))
    keys = orc.keygen(P, seed=2100, rotations=rots)

    def enc(t, part, lvl, idx):
        v = np.concatenate([radar.pack_vital(getattr(scenes[s][t], part), n) for s in range(S)])
        return orc.encrypt(P, keys, orc.encode(P, v, float(2 ** P.scale_bits), lvl), lvl, float(2 ** P.scale_bits),
                           n, seed=31, index=idx)

    # V1 at level 3
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    re = [enc(t, "real", 3, 2 * t) for t in range(F)]
    im = [enc(t, "imag", 3, 2 * t + 1) for t in range(F)]
    Nc, Dc = cc.vitals_v1(ev, cc.PlainBook(P), re, im, cfg)
    assert ("relin_rescale" in [op for op, _, _ in ev.trace]) == bool(merge)  # R31 on the vital chains
    Nd, Dd = _decode_all(P, keys, Nc), _decode_all(P, keys, Dc)
    for s in range(S):
        Np, Dp, _ = dsp.soft_attention(dsp.energy(scenes[s]), cfg.gamma, F)
        assert abs(Nd[s * n] - Np) <= 1e-3 * abs(Np) and abs(Dd[s * n] - Dp) <= 1e-3 * abs(Dp), s
    # V2 at level 7
    ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
    re = [enc(t, "real", 7, 2 * t) for t in range(F)]
    im = [enc(t, "imag", 7, 2 * t + 1) for t in range(F)]
    taps = [np.array([0.2, 0.3, 0.3, 0.2]), np.array([0.25, -0.5, 0.25])]
    out = cc.vitals_v2(ev, re, im, taps, cfg)
    for s in range(S):
        I = np.array([dsp.soft_iq(scenes[s][t], cfg.p_phi)[0] for t in range(F)])
        Q = np.array([dsp.soft_iq(scenes[s][t], cfg.p_phi)[1] for t in range(F)])
        for bi, h in enumerate(taps):
            y = dsp.taylor_phase(dsp.fir(I, h), dsp.fir(Q, h), cfg.taylor_order)
            want = dsp.narrowband_power(y, dsp.band_bins(len(y), cfg.fs, cfg.bands[bi]))
            got = np.array([_decode_all(P, keys, c)[s * n] for c in out[bi]])
            assert rel_err(got, want) < 1e-3, (s, bi)
