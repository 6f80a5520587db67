"""GPU parity: every CUDA primitive and chain, called through the C-ABI, must
reproduce the CPU oracle's residues bit for bit (north_star gate 1), with
equal op traces (Theorem P:999-1006).  Inputs are seeded: oracle keys and
encryptions, or uniform residues (the ciphertext distribution) where only the
arithmetic is under test."""
import numpy as np
import pytest

from oracle import ckks as orc
from oracle import circuits as cc
from synth import prng
from synth.params import ps1, ps3, ps4, toy

from gpu_util import ct_in, ct_out, dev_tensor, host, make_ctx, residues, uniform_poly

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m(cuda_ctx_ok):
    from paper_2603_22437_b200 import build, mmfhe
    build.build()
    return mmfhe


def _rand_ct(P, level, seed):
    c = uniform_poly(P, level, seed, prng.SID_UNIFORM, 2)
    return orc.Ct([c[0], c[1]], level, float(2 ** P.scale_bits), P.n // 2)


# ------------------------------------------------------------------ NTT / products

@pytest.mark.parametrize("log_n", [5, 10, 13, 14, 15, 16])
def test_ntt_roundtrip_and_negacyclic_product(m, log_n):
    P = toy(log_n=log_n, n_q=3, scale_bits=50, n_p=1, alpha=1)
    ctx = make_ctx(m, P)
    rows = uniform_poly(P, 2, 11, prng.SID_UNIFORM, 1)[0]
    d = dev_tensor(rows)
    ctx.ntt(d, [0, 1, 2])
    assert not np.array_equal(host(d), rows)
    ctx.ntt(d, [0, 1, 2], inverse=True)
    assert np.array_equal(host(d), rows)
    # pmult = negacyclic ring product per limb (NTT, Montgomery product, INTT)
    a = _rand_ct(P, 2, 12)
    b = uniform_poly(P, 2, 13, prng.SID_UNIFORM + 7, 1)[0]
    ctx.load_plain("b", b, 2, 1.0)
    out = ct_out(m, P, 2)
    ctx.pmult(ct_in(m, P, a), "b", out)
    got = residues(out)
    qs = list(P.q[:3])
    assert np.array_equal(got[0], orc.poly_mul(qs, a.c[0], b))
    assert np.array_equal(got[1], orc.poly_mul(qs, a.c[1], b))


def test_host_buffers_roundtrip(m):
    P = toy(log_n=10, n_q=3)
    ctx = make_ctx(m, P)
    a, b = _rand_ct(P, 2, 1), _rand_ct(P, 2, 2)
    out = ct_out(m, P, 2, device=False)
    ctx.hadd(ct_in(m, P, a, device=False), ct_in(m, P, b, device=False), out)
    qs = list(P.q[:3])
    assert np.array_equal(out.data[0], orc.poly_add(qs, a.c[0], b.c[0]))
    assert np.array_equal(out.data[1], orc.poly_add(qs, a.c[1], b.c[1]))
    ctx.hsub(ct_in(m, P, a, device=False), ct_in(m, P, b, device=False), out)
    assert np.array_equal(out.data[0], orc.poly_sub(qs, a.c[0], b.c[0]))


# ------------------------------------------------------------------ rescale / KS / HRot / HMult

@pytest.mark.parametrize("level", [1, 2, 5])
def test_rescale_parity(m, level):
    P = toy(log_n=11, n_q=6, scale_bits=40, n_p=2, alpha=2)
    ctx = make_ctx(m, P)
    a = _rand_ct(P, level, 20 + level)
    ev = orc.Evaluator(P)
    want = ev.rescale(a)
    out = ct_out(m, P, level - 1)
    ctx.rescale(ct_in(m, P, a), out)
    assert np.array_equal(residues(out), np.stack(want.c))
    assert out.level == want.level and out.scale == want.scale


@pytest.fixture(scope="module")
def toy_keys():
    P = toy(log_n=11, n_q=6, scale_bits=40, n_p=2, alpha=2)
    return P, orc.keygen(P, seed=501, rotations=[1, 3, -1, 100])


@pytest.mark.parametrize("level", [5, 4, 2, 0])
def test_keyswitch_parity(m, toy_keys, level):
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    x = uniform_poly(P, level, 40 + level, prng.SID_UNIFORM, 1)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    d0, d1 = ev.keyswitch(x[0], level, keys.rlk)
    out = ct_out(m, P, level)
    ctx.keyswitch(m.Ct(dev_tensor(x), level, 1.0, 0, P.log_n, m.FORM_COEFF, 1), out, use_relin=True)
    got = residues(out)
    assert np.array_equal(got[0], d0) and np.array_equal(got[1], d1)


@pytest.mark.parametrize("step,level", [(1, 5), (3, 3), (-1, 5), (100, 1), (1, 0)])
def test_hrot_parity(m, toy_keys, step, level):
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, level, 60 + step % 97 + level)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    want = ev.rotate(a, step)
    out = ct_out(m, P, level)
    ctx.hrot(ct_in(m, P, a), step, out)
    assert np.array_equal(residues(out), np.stack(want.c))
    assert ctx.trace() == ev.trace


@pytest.mark.parametrize("level", [5, 3, 0])
def test_hrot_hoisted_parity(m, toy_keys, level):
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, level, 65 + level)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    steps = [1, 3, -1, 100, 0]
    want = ev.rotate_hoisted(a, steps)
    outs = [ct_out(m, P, level) for _ in steps]
    ctx.hrot_hoisted(ct_in(m, P, a), steps, outs)
    for o, w in zip(outs, want):
        assert np.array_equal(residues(o), np.stack(w.c))
    assert ctx.trace() == ev.trace


def _pq_want(ct):
    """Oracle PQ ciphertext (coefficient form over q_0..q_l, p_0..p_{K-1} per poly) in the
    library's PQ layout: Q rows of poly 0 / poly 1, then P rows of poly 0 / poly 1."""
    l1 = ct.level + 1
    return np.concatenate([ct.c[0][:l1], ct.c[1][:l1], ct.c[0][l1:], ct.c[1][l1:]])


def _pq_out(m, P, level):
    import torch
    data = torch.empty((2 * (level + 1 + P.K), P.n), dtype=torch.int64, device="cuda:0")
    return m.Ct(data, level, 0.0, 0, P.log_n, m.FORM_COEFF, 2)


@pytest.mark.parametrize("level", [5, 2])
def test_hrot_hoisted_pq_parity(m, toy_keys, level):
    """Double hoisting's baby steps through mmfhe_hrot_hoisted_pq (the PQ lift for step 0):
    residues equal the oracle's lift_pq / hoisted_step_pq."""
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, level, 75 + level)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    steps = [0, 1, 3, -1, 100]
    ys = ev.hoist_modup(a)
    want = [ev.hoisted_step_pq(a, ys, s) for s in steps]
    outs = [_pq_out(m, P, level) for _ in steps]
    ctx.hrot_hoisted_pq(ct_in(m, P, a), steps, outs)
    for o, w in zip(outs, want):
        assert np.array_equal(residues(o), _pq_want(w))


@pytest.mark.parametrize("level", [5, 0])
def test_conjugation_parity(m, toy_keys, level):
    """Conj (DESIGN R28) through the HRot primitive with MMFHE_STEP_CONJ: residues and trace
    equal the oracle's Evaluator.conjugate (key from the oracle keygen's CONJ entry)."""
    P, _ = toy_keys
    keys = orc.keygen(P, seed=1777, rotations=[orc.CONJ])
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, level, 85 + level)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    want = ev.conjugate(a)
    out = ct_out(m, P, level)
    ctx.hrot(ct_in(m, P, a), m.STEP_CONJ, out)
    assert np.array_equal(residues(out), np.stack(want.c))
    assert ctx.trace() == ev.trace == [("conj", level, "")]


@pytest.mark.parametrize("level", [5, 2])
def test_hmult_relin_parity(m, toy_keys, level):
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    a, b = _rand_ct(P, level, 70), _rand_ct(P, level, 71)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    want = ev.mul_relin(a, b)
    out = ct_out(m, P, level)
    ctx.hmult(ct_in(m, P, a), ct_in(m, P, b), out)
    assert np.array_equal(residues(out), np.stack(want.c))
    assert out.scale == want.scale
    # relin of an explicit 3-poly tensor
    t = ev.tensor(a, a)
    out3 = ct_out(m, P, level)
    ctx.relin(ct_in(m, P, t), out3)
    assert np.array_equal(residues(out3), np.stack(ev.relin(t).c))


def test_mod_switch_and_sum_partials(m, toy_keys):
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    cts = [_rand_ct(P, 4, 80 + i) for i in range(5)]
    ev = orc.Evaluator(P)
    want = cts[0]
    for c in cts[1:]:
        want = ev.add(want, c)
    out = ct_out(m, P, 4)
    ctx.sum_partials([ct_in(m, P, c) for c in cts], out)
    assert np.array_equal(residues(out), np.stack(want.c))
    out2 = ct_out(m, P, 2)
    ctx.mod_switch(ct_in(m, P, cts[0]), 2, out2)
    assert np.array_equal(residues(out2), np.stack([c[:3] for c in cts[0].c]))


def test_errors(m, toy_keys):
    P, keys = toy_keys
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, 0, 90)
    with pytest.raises(m.MmfheError) as e:
        ctx.rescale(ct_in(m, P, a), ct_out(m, P, 0))
    assert e.value.name == "E_DEPTH"
    with pytest.raises(m.MmfheError) as e:
        ctx.hrot(ct_in(m, P, _rand_ct(P, 3, 91)), 7, ct_out(m, P, 3))
    assert e.value.name == "E_MISSING_KEY"
    b = _rand_ct(P, 3, 92)
    b.scale *= 2
    with pytest.raises(m.MmfheError) as e:
        ctx.hadd(ct_in(m, P, _rand_ct(P, 3, 93)), ct_in(m, P, b), ct_out(m, P, 3))
    assert e.value.name == "E_SCALE"
    with pytest.raises(m.MmfheError) as e:
        m.Context(10, [97], [193], 1, 40)
    assert e.value.name == "E_PARAMS"


# ------------------------------------------------------------------ full-size (PS4, N = 2^16)

@pytest.fixture(scope="module")
def ps4_keys():
    P = ps4()
    return P, orc.keygen(P, seed=4001, rotations=[1, 5, 2048])


@pytest.mark.parametrize("step", [1, 2048])
def test_ps4_hrot_parity(m, ps4_keys, step):
    P, keys = ps4_keys
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, P.L, 4100 + step)
    want = orc.Evaluator(P, keys.rlk, keys.gk).rotate(a, step)
    out = ct_out(m, P, P.L)
    ctx.hrot(ct_in(m, P, a), step, out)
    assert np.array_equal(residues(out), np.stack(want.c))


def test_ps4_hmult_rescale_parity(m, ps4_keys):
    P, keys = ps4_keys
    ctx = make_ctx(m, P, keys)
    a, b = _rand_ct(P, P.L, 4200), _rand_ct(P, P.L, 4201)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    want = ev.mul_relin(a, b)
    out = ct_out(m, P, P.L)
    ctx.hmult(ct_in(m, P, a), ct_in(m, P, b), out)
    assert np.array_equal(residues(out), np.stack(want.c))
    want_r = ev.rescale(want)
    out_r = ct_out(m, P, P.L - 1)
    ctx.rescale(out, out_r)
    assert np.array_equal(residues(out_r), np.stack(want_r.c))


def test_ps4_hrot_hoisted_pq_parity(m, ps4_keys):
    """The bench's evk-streaming step at N = 2^16 (PS4 top level, 3 digits: the grouped inner
    product k_hoisted_ip_pq): PQ baby steps bit-exact against the oracle."""
    P, keys = ps4_keys
    ctx = make_ctx(m, P, keys)
    a = _rand_ct(P, P.L, 4300)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    steps = [1, 5, 2048]
    ys = ev.hoist_modup(a)
    want = [ev.hoisted_step_pq(a, ys, s) for s in steps]
    outs = [_pq_out(m, P, P.L) for _ in steps]
    ctx.hrot_hoisted_pq(ct_in(m, P, a), steps, outs)
    for o, w in zip(outs, want):
        assert np.array_equal(residues(o), _pq_want(w))
