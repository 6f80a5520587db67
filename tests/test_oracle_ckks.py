"""Pins for the O-RNS CKKS layer: encode/encrypt round trips,
the automorphism slot-rotation invariant, homomorphic add/mult/rotate against
plain slot-wise arithmetic, the chained-squaring error bound of P:1049-1055,
and the exact scalar-constant encoding."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import ckks as orc
from synth.params import toy


@pytest.fixture(scope="module")
def P():
    return toy(log_n=10, n_q=6, scale_bits=40, n_p=2, alpha=2)


@pytest.fixture(scope="module")
def keys(P):
    return orc.keygen(P, seed=123, rotations=[1, 2, 3, 5, -1, 64])


def test_embedding_roundtrip(P):
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, P.n // 2)
    m = orc.embed_inverse(v, P.n)
    assert np.max(np.abs(orc.embed(m, P.n).real - v)) < 1e-12
    assert np.max(np.abs(orc.embed(m, P.n).imag)) < 1e-12


def test_embedding_is_evaluation_at_roots():
    # z_j = m(zeta^(5^j mod 2N)) written out directly at N=16
    n = 16
    rng = np.random.default_rng(1)
    m = rng.normal(size=n)
    z = orc.embed(m, n)
    for j in range(n // 2):
        root = np.exp(1j * np.pi * pow(5, j, 2 * n) / n)
        assert abs(np.polyval(m[::-1], root) - z[j]) < 1e-9


@pytest.mark.parametrize("k", [1, 3, -2, 5])
def test_automorphism_rotates_slots(k):
    # decode(sigma_{5^k}(encode(v))) = roll(v, -k)
    n = 32
    rng = np.random.default_rng(k + 10)
    v = rng.uniform(-1, 1, n // 2)
    m = np.rint(orc.embed_inverse(v, n) * 2 ** 30).astype(np.int64)
    g = pow(5, k % (n // 2), 2 * n)
    out = np.zeros(n)
    for i, x in enumerate(m):
        j = i * g % (2 * n)
        if j < n:
            out[j] += x
        else:
            out[j - n] -= x
    z = orc.embed(out / 2 ** 30, n).real
    assert np.max(np.abs(z - np.roll(v, -k))) < 1e-6


def test_encrypt_decrypt_roundtrip(P, keys):
    rng = np.random.default_rng(2)
    v = rng.uniform(-1, 1, 128)
    ct = orc.encrypt_vector(P, keys, v, P.L, seed=5, index=0)
    out = orc.decrypt_vector(P, keys, ct)
    assert np.max(np.abs(out - v)) < 2 ** -20


def test_hadd_hmult_rotate(P, keys):
    rng = np.random.default_rng(3)
    n = 128
    a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    ca = orc.encrypt_vector(P, keys, a, P.L, seed=6, index=0)
    cb = orc.encrypt_vector(P, keys, b, P.L, seed=6, index=1)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    s = orc.decrypt_vector(P, keys, ev.add(ca, cb))
    assert np.max(np.abs(s - (a + b))) < 2 ** -20
    m = ev.mul_rescale(ca, cb)
    assert m.level == P.L - 1
    assert np.max(np.abs(orc.decrypt_vector(P, keys, m) - a * b)) < 2 ** -18
    for k in (1, 3, -1, 64):
        r = ev.rotate(ca, k)
        assert np.max(np.abs(orc.decrypt_vector(P, keys, r) - np.roll(a, -k))) < 2 ** -20
    # Rot(Enc([0,1,2,...]),1) -> [1,2,...,0]
    ramp = np.arange(n) / n
    cr = orc.encrypt_vector(P, keys, ramp, P.L, seed=6, index=2)
    assert np.max(np.abs(orc.decrypt_vector(P, keys, ev.rotate(cr, 1)) - np.roll(ramp, -1))) < 2 ** -20


def test_hoisted_rotation(P, keys):
    # hoisted HRot decrypts to the rotation, but is a different op:
    # BConv does not commute with sigma_g's sign flips, so residues differ from rotate()
    rng = np.random.default_rng(9)
    n = 128
    a = rng.uniform(-1, 1, n)
    ca = orc.encrypt_vector(P, keys, a, P.L, seed=8, index=0)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    outs = ev.rotate_hoisted(ca, [1, 3, -1, 64, 0])
    for k, c in zip([1, 3, -1, 64], outs):
        assert np.max(np.abs(orc.decrypt_vector(P, keys, c) - np.roll(a, -k))) < 2 ** -20
    assert outs[4] is ca
    plain = ev.rotate(ca, 3)
    assert not np.array_equal(np.stack(plain.c), np.stack(outs[1].c))
    assert [t for t in ev.trace if t[0] == "hrot_hoisted"] == [("hrot_hoisted", P.L, s) for s in
                                                               ("1", "3", str(P.n // 2 - 1), "64")]
    # lower level: digits truncated at level l (SURVEY c-5 "Keys")
    low = orc.Ct([x[:3].copy() for x in ca.c], 2, ca.scale, ca.n_slots)
    r = ev.rotate_hoisted(low, [5])[0]
    assert np.max(np.abs(orc.decrypt_vector(P, keys, r) - np.roll(a, -5))) < 2 ** -20


def test_plain_mult_and_scalar(P, keys):
    rng = np.random.default_rng(4)
    n = 128
    a, w = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    ca = orc.encrypt_vector(P, keys, a, P.L, seed=7, index=0)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    ql = P.q[P.L]
    pt = orc.encode(P, w, ql, P.L)
    r = ev.rescale(ev.pmult(ca, pt, ql))
    assert r.scale == ca.scale  # PMult at Delta_pt = q_l preserves scale exactly (c-6)
    assert np.max(np.abs(orc.decrypt_vector(P, keys, r) - a * w)) < 2 ** -20
    r2 = ev.rescale(ev.pmult_scalar(ca, -1.0 / 3.0))
    assert np.max(np.abs(orc.decrypt_vector(P, keys, r2) + a / 3)) < 2 ** -20


def test_chained_squarings_error(keys):
    # cumulative rescale error ~ L * 2^-Delta; S:139 -- 11 squarings of Enc(0.9)
    # hybrid KS needs P >= the largest digit product: alpha=2 digits (<= 100 bits) vs P ~ 2^120
    P = toy(log_n=10, n_q=12, scale_bits=40, n_p=2, alpha=2)
    k = orc.keygen(P, seed=77)
    ev = orc.Evaluator(P, k.rlk)
    x = np.linspace(0.9999, 0.99995, 16)  # x^(2^11) stays O(1)
    ct = orc.encrypt_vector(P, k, x, P.L, seed=8, index=0)
    want = x.copy()
    for _ in range(11):
        ct = ev.square_rescale(ct)
        want = want * want
    assert ct.level == 0
    got = orc.decrypt_vector(P, k, ct)
    # relative error bounded by 2^11 amplification of the fresh error (~2^-30)
    assert np.max(np.abs(got - want) / np.abs(want)) < 1e-4
    with pytest.raises(orc.DepthError):
        ev.rescale(ev.relin(ev.tensor(ct, ct)))


@pytest.mark.parametrize("c", [0.5, -0.5, 1 / 3, -1 / 3, 2.5e-7, 0.1, -0.75, 1.0])
def test_scalar_encoding_exact(c):
    q = (1 << 60) - 93  # any 60-bit odd modulus
    v = orc.encode_scalar(c, q)
    exact = Fraction(c) * q
    assert abs(Fraction(v) - exact) <= Fraction(1, 2)
    if abs(Fraction(v) - exact) == Fraction(1, 2):
        assert abs(v) > abs(exact)  # ties away from zero


def test_missing_key_and_scale_errors(P, keys):
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    ct = orc.encrypt_vector(P, keys, np.zeros(8), P.L, seed=1, index=0)
    with pytest.raises(KeyError):
        ev.rotate(ct, 7)
    ct2 = orc.Ct([c.copy() for c in ct.c], ct.level, ct.scale * 2, ct.n_slots)
    with pytest.raises(orc.ScaleError):
        ev.add(ct, ct2)


def test_evk_sizes_match_paper():
    # vital relin key 22.5 MiB = dnum 3 x 2 x (11 Q + 4 P) limbs x 2^15 x 8 B
    from synth.params import make_params
    P = make_params(15, 11, 40, 4, 4, name="vital-paper")
    assert P.dnum() == 3
    size = P.dnum() * 2 * (len(P.q) + len(P.p)) * P.n * 8
    assert size / 2 ** 20 == pytest.approx(22.5)
    # ciphertext 5.5 MiB = 2 x 11 limbs x 2^15 x 8 B
    assert 2 * len(P.q) * P.n * 8 / 2 ** 20 == pytest.approx(5.5)


def test_paper_vital_parameter_set_reproduces_published_sizes():
    """PSV: N=2^15, 11 Q limbs (60 + 10 x 40 bits), dnum 3 with
    K = alpha = 4 special primes reproduces the paper's 5.5 MB ciphertext and 22.5 MB
    relinearisation key (Table tab:comm_overhead), within the 128-bit HE-standard bound
    for N = 2^15 (log2 PQ <= 881)."""
    from synth.params import psv
    P = psv()
    MiB = 2 ** 20
    assert 2 * len(P.q) * P.n * 8 / MiB == 5.5
    assert P.dnum() * 2 * (len(P.q) + len(P.p)) * P.n * 8 / MiB == 22.5
    assert sum(q.bit_length() for q in P.q + P.p) <= 881
    assert all((q - 1) % (2 * P.n) == 0 for q in P.q + P.p)


# ------------------------------------------------------------------ complex slots (reading R28)

def test_complex_embedding_is_evaluation_at_roots():
    """A complex slot vector z encodes to REAL coefficients m with m(zeta^(5^j)) = z_j (the
    polynomial evaluated directly at the roots, N = 16), and m(zeta^(-5^j)) = conj z_j."""
    n = 16
    rng = np.random.default_rng(3)
    z = rng.normal(size=n // 2) + 1j * rng.normal(size=n // 2)
    m = orc.embed_inverse(z, n)
    assert m.dtype.kind == "f"
    for j in range(n // 2):
        e = pow(5, j, 2 * n)
        assert abs(np.polyval(m[::-1], np.exp(1j * np.pi * e / n)) - z[j]) < 1e-9
        assert abs(np.polyval(m[::-1], np.exp(-1j * np.pi * e / n)) - np.conj(z[j])) < 1e-9


def test_conjugation_automorphism_conjugates_slots():
    """sigma_{2N-1} (X -> X^-1 = -X^(N-1)) applied to the coefficients written out by hand
    conjugates every slot (N = 32), and orc.galois_element maps CONJ to 2N - 1."""
    n = 32
    P = toy(log_n=5, n_q=2, scale_bits=30, n_p=1, alpha=2)
    assert orc.galois_element(P, orc.CONJ) == 2 * n - 1
    rng = np.random.default_rng(4)
    z = rng.uniform(-1, 1, n // 2) + 1j * rng.uniform(-1, 1, n // 2)
    m = np.rint(orc.embed_inverse(z, n) * 2 ** 30).astype(np.int64)
    out = np.zeros(n)
    out[0] = m[0]
    out[1:] = -m[1:][::-1]  # X^i -> X^(-i) = -X^(N-i)
    got = orc.embed(out / 2 ** 30, n)
    assert np.max(np.abs(got - np.conj(z))) < 1e-6


def test_complex_slots_encrypted(P):
    """Complex slot vectors through the evaluator: encrypt -> decrypt, Conj (the conjugation
    key switch), rotation, and the slot-wise complex product z w and z conj(z) = |z|^2."""
    keys = orc.keygen(P, seed=321, rotations=[3, orc.CONJ])
    assert orc.CONJ in keys.gk and 3 in keys.gk
    rng = np.random.default_rng(9)
    h = P.n // 2
    z = rng.uniform(-1, 1, h) + 1j * rng.uniform(-1, 1, h)
    w = rng.uniform(-1, 1, h) + 1j * rng.uniform(-1, 1, h)
    lvl = P.L
    cz = orc.encrypt_vector(P, keys, z, lvl, seed=5, index=0)
    cw = orc.encrypt_vector(P, keys, w, lvl, seed=5, index=1)
    dec = orc.decrypt_vector(P, keys, cz, complex_out=True)
    assert np.max(np.abs(dec - z)) < 1e-6
    assert np.max(np.abs(orc.decrypt_vector(P, keys, cz) - z.real)) < 1e-6
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    cj = ev.conjugate(cz)
    assert ev.trace[-1] == ("conj", lvl, "")
    assert np.max(np.abs(orc.decrypt_vector(P, keys, cj, complex_out=True) - np.conj(z))) < 1e-6
    r = ev.rotate(cz, 3)
    assert np.max(np.abs(orc.decrypt_vector(P, keys, r, complex_out=True) - np.roll(z, -3))) < 1e-6
    zw = ev.mul_rescale(cz, cw)
    assert np.max(np.abs(orc.decrypt_vector(P, keys, zw, complex_out=True) - z * w)) < 1e-5
    p = orc.decrypt_vector(P, keys, ev.mul_rescale(cz, cj), complex_out=True)
    assert np.max(np.abs(p.real - np.abs(z) ** 2)) < 1e-5 and np.max(np.abs(p.imag)) < 1e-5
    with pytest.raises(KeyError):
        orc.Evaluator(P, keys.rlk, {3: keys.gk[3]}).conjugate(cz)


def test_real_encoding_unchanged_by_complex_support(P):
    """A real vector and the same vector as complex with zero imaginary parts encode to the
    same integers (the real path is the complex path's special case)."""
    rng = np.random.default_rng(11)
    v = rng.uniform(-1, 1, 64)
    a = orc.encode(P, v, 2.0 ** 30, 1)
    b = orc.encode(P, v.astype(np.complex128), 2.0 ** 30, 1)
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ merged ModDown + rescale (reading R31)

def test_relin_rescale_merged_and_moddown_rescale(P, keys):
    """Reading R31: relinearisation + rescale as one division by P q_l decrypts to the product like
    mul_rescale (scale, level, values), and the PQ lift brought down by the merged division equals
    the rescaled ciphertext's message; the trace records the merged ops."""
    rng = np.random.default_rng(21)
    h = P.n // 2
    a = rng.uniform(-1, 1, h)
    b = rng.uniform(-1, 1, h)
    lvl = P.L
    ca = orc.encrypt_vector(P, keys, a, lvl, seed=7, index=0)
    cb = orc.encrypt_vector(P, keys, b, lvl, seed=7, index=1)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    t = ev.tensor(ca, cb)
    m = ev.relin_rescale_merged(t)
    r = ev.mul_rescale(ca, cb)
    assert m.level == r.level == lvl - 1 and m.scale == r.scale
    assert ev.trace[1] == ("relin_rescale", lvl, "")
    assert np.max(np.abs(orc.decrypt_vector(P, keys, m) - a * b)) < 1e-5
    assert np.max(np.abs(orc.decrypt_vector(P, keys, m) - orc.decrypt_vector(P, keys, r))) < 1e-6
    rl = ev.relin(t)  # scale Delta^2: the PQ lift of it divided by P q_l is the rescaled product
    d = ev.moddown_rescale_ct(ev.lift_pq(rl))
    assert d.level == lvl - 1 and d.scale == rl.scale / P.q[lvl]
    assert np.max(np.abs(orc.decrypt_vector(P, keys, d) - a * b)) < 1e-5
    assert np.max(np.abs(orc.decrypt_vector(P, keys, d) - orc.decrypt_vector(P, keys, ev.rescale(rl)))) < 1e-6


def test_conj_mul_relin_rescale(P):
    """Reading R32: d Conj(d) with the conjugation and conjugate-product keys and one division by
    P q_l decrypts to |d|^2 (complex slots), equals the two-key-switch path to the noise level, and
    the key set / trace are as stated."""
    keys = orc.keygen(P, seed=654, rotations=[orc.CONJ, orc.CONJ_PROD])
    assert orc.CONJ in keys.gk and orc.CONJ_PROD in keys.gk
    rng = np.random.default_rng(31)
    h = P.n // 2
    z = rng.uniform(-1, 1, h) + 1j * rng.uniform(-1, 1, h)
    lvl = P.L
    cz = orc.encrypt_vector(P, keys, z, lvl, seed=9, index=0)
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    f = ev.conj_mul_relin_rescale(cz)
    assert ev.trace == [("conj_mul_relin_rescale", lvl, "")]
    assert f.level == lvl - 1 and f.scale == cz.scale * cz.scale / P.q[lvl]
    got = orc.decrypt_vector(P, keys, f, complex_out=True)
    assert np.max(np.abs(got.real - np.abs(z) ** 2)) < 1e-5 and np.max(np.abs(got.imag)) < 1e-5
    two = ev.relin_rescale_merged(ev.tensor(cz, ev.conjugate(cz)))
    assert np.max(np.abs(orc.decrypt_vector(P, keys, two) - got.real)) < 1e-5
    with pytest.raises(KeyError):
        orc.Evaluator(P, keys.rlk, {orc.CONJ: keys.gk[orc.CONJ]}).conj_mul_relin_rescale(cz)
