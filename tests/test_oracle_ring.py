"""Pins for O-RNS ring arithmetic against O-BIG and mathematics.

Each test would fail on a plausible mistake in ckks_ref.c: a wrong twist or
root order (NTT round trip / schoolbook product), a dropped negacyclic sign
(X*X^(N-1) = -1), a wrong automorphism sign, an off-by-one in the rescale
rounding (exact CRT comparison), a missing ModUp/ModDown term (big-int
invariants).
"""
import random

import numpy as np
import pytest

from oracle import bigint_ref as big
from oracle import ckks as orc
from synth.params import is_prime, primes_below, toy


def _rand_res(rng, qs, n):
    return np.stack([np.array([rng.randrange(q) for _ in range(n)], dtype=np.uint64) for q in qs])


@pytest.mark.parametrize("n", [8, 16, 64])
def test_negacyclic_product_matches_schoolbook(n):
    rng = random.Random(n)
    qs = primes_below(1 << 60, 2 * n, 2) + primes_below(1 << 30, 2 * n, 1)
    a = _rand_res(rng, qs, n)
    b = _rand_res(rng, qs, n)
    got = orc.poly_mul(qs, a, b)
    for l, q in enumerate(qs):
        want = big.schoolbook_negacyclic([int(x) for x in a[l]], [int(x) for x in b[l]], q)
        assert [int(x) for x in got[l]] == want


def test_x_times_x_pow_n_minus_1_is_minus_one():
    # X * X^(N-1) = X^N = -1 in Z_q[X]/(X^N+1)
    n = 32
    q = primes_below(1 << 60, 2 * n, 1)[0]
    a = np.zeros((1, n), dtype=np.uint64); a[0, 1] = 1
    b = np.zeros((1, n), dtype=np.uint64); b[0, n - 1] = 1
    c = orc.poly_mul([q], a, b)
    want = np.zeros(n, dtype=np.uint64); want[0] = q - 1
    assert np.array_equal(c[0], want)


@pytest.mark.parametrize("log_n", [4, 10, 13])
def test_ntt_roundtrip_and_evaluation(log_n):
    n = 1 << log_n
    q = primes_below(1 << 60, 2 * n, 1)[0]
    rng = np.random.default_rng(log_n)
    a = (rng.integers(0, 1 << 62, n, dtype=np.uint64) % np.uint64(q)).astype(np.uint64)
    x = a.copy()
    lib = orc.lib()
    assert lib.or_ntt_forward(n, q, x) == 0
    # NTT output k is a(psi^(2k+1)): check a few points by Horner with big ints
    psi = lib.or_find_psi(q, n)
    assert pow(psi, n, q) == q - 1
    for k in (0, 1, n // 2, n - 1):
        r = pow(psi, 2 * k + 1, q)
        v = 0
        for c in reversed(a.tolist()):
            v = (v * r + c) % q
        assert int(x[k]) == v
    assert lib.or_ntt_inverse(n, q, x) == 0
    assert np.array_equal(x, a)


def test_constant_poly_ntt_is_constant():
    n = 64
    q = primes_below(1 << 60, 2 * n, 1)[0]
    a = np.zeros(n, dtype=np.uint64); a[0] = 12345
    orc.lib().or_ntt_forward(n, q, a)
    assert np.all(a == 12345)


@pytest.mark.parametrize("g", [5, 25, 3, 2 * 32 - 1])
def test_automorphism_matches_bigint(g):
    n = 32
    qs = primes_below(1 << 60, 2 * n, 2)
    rng = random.Random(g)
    a = [rng.randrange(-1000, 1000) for _ in range(n)]
    res = orc.small_to_rns(np.array(a), qs)
    got = orc.automorphism(qs, res, g)
    want = big.galois_apply(a, g)
    for l, q in enumerate(qs):
        assert [int(x) for x in got[l]] == [w % q for w in want]


def test_automorphism_is_ring_homomorphism():
    # sigma_g(a*b) = sigma_g(a) * sigma_g(b)
    n = 64
    qs = primes_below(1 << 60, 2 * n, 1)
    rng = random.Random(7)
    a = _rand_res(rng, qs, n)
    b = _rand_res(rng, qs, n)
    g = 5 ** 3 % (2 * n)
    lhs = orc.automorphism(qs, orc.poly_mul(qs, a, b), g)
    rhs = orc.poly_mul(qs, orc.automorphism(qs, a, g), orc.automorphism(qs, b, g))
    assert np.array_equal(lhs, rhs)


def _small_chain(n, n_q, bits_q=22, n_p=2, bits_p=25):
    two_n = 2 * n
    qs = primes_below(1 << bits_q, two_n, n_q)
    ps = primes_below(1 << bits_p, two_n, n_p)
    return qs, ps


def test_rescale_equals_round_half_up_of_crt():
    # rescale == round-half-up(A / q_l) mod Q_{l-1}, 2000 CRT integers
    n = 16
    qs, _ = _small_chain(n, 5)
    rng = random.Random(11)
    l = len(qs) - 1
    for _ in range(2000 // n):
        a = _rand_res(rng, qs, n)
        # include exact ties: force some coefficients to A = k*q_l + floor(q_l/2)
        out = np.empty((l, n), dtype=np.uint64)
        orc.lib().or_rescale(n, l, orc._arr(qs), orc._arr(a), out)
        A, Q = big.crt([a[i] for i in range(l + 1)], qs)
        Qm = Q // qs[l]
        for k in range(n):
            want = big.round_half_up_div(A[k], qs[l]) % Qm
            got, _ = big.crt([out[i][k:k + 1] for i in range(l)], qs[:l])
            assert got[0] == want


def test_rescale_ties_round_up():
    n = 16
    qs, _ = _small_chain(n, 3)
    l = 2
    ql = qs[l]
    Qm = qs[0] * qs[1]
    # A = k*q_l + floor(q_l/2) + 1 (q_l odd -> exactly .5 above k*q_l + q_l/2 - 0.5)
    vals = [k * ql + ql // 2 + 1 for k in range(n)] + [k * ql + ql // 2 for k in range(n)]
    for chunk in (vals[:n], vals[n:]):
        a = np.stack([np.array([v % q for v in chunk], dtype=np.uint64) for q in qs])
        out = np.empty((l, n), dtype=np.uint64)
        orc.lib().or_rescale(n, l, orc._arr(qs), orc._arr(a), out)
        got, _ = big.crt([out[0], out[1]], qs[:2])
        assert got == [big.round_half_up_div(v, ql) % Qm for v in chunk]


def test_modup_invariant():
    # CRT(y_j) - x_j in {0..|I_j|-1} * Q_j
    n = 16
    qs, ps = _small_chain(n, 5)
    alpha = 2
    rng = random.Random(3)
    for l in (4, 3, 2):
        x = _rand_res(rng, qs[: l + 1], n)
        for j in range(-(-(l + 1) // alpha)):
            lo, hi = j * alpha, min(j * alpha + alpha, l + 1)
            y = np.empty((l + 1 + len(ps), n), dtype=np.uint64)
            orc.lib().or_modup(n, l, orc._arr(qs), len(ps), orc._arr(ps), alpha, j, orc._arr(x), y)
            basis = qs[: l + 1] + ps
            Y, _ = big.crt([y[t] for t in range(len(basis))], basis)
            X, Qj = big.crt([x[t] for t in range(lo, hi)], qs[lo:hi])
            for k in range(n):
                d = Y[k] - X[k]
                assert d % Qj == 0 and 0 <= d // Qj < hi - lo


def test_moddown_is_division_by_p_within_k():
    # ModDown(c') = (c' - BConv_P(c'_P)) / P: result*P - c' == -(c'_P + u P), so
    # |result - c'/P| <= K (fast BConv error u in [0, K)); exactness: result*P = c' - w mod Q
    n = 16
    qs, ps = _small_chain(n, 4)
    l = 3
    rng = random.Random(5)
    basis = qs + ps
    c = _rand_res(rng, basis, n)
    out = np.empty((l + 1, n), dtype=np.uint64)
    orc.lib().or_moddown(n, l, orc._arr(qs), len(ps), orc._arr(ps), orc._arr(c), out)
    C, QP = big.crt([c[t] for t in range(len(basis))], basis)
    R, Q = big.crt([out[t] for t in range(l + 1)], qs)
    P = ps[0] * ps[1]
    for k in range(n):
        cc = big.centered(C[k], QP)
        rr = big.centered(R[k], Q)
        assert abs(rr * P - cc) <= (len(ps) + 1) * P


def test_moddown_rescale_is_division_by_p_ql_within_k1():
    # Reading R31: the merged ModDown + rescale is (c' - BConv_{P u q_l}(c')) / (P q_l); with the
    # big-integer CRT value C of c' over Q_l u P and R of the result over Q_{l-1}:
    # R = (C - [C]_{P q_l} - u P q_l) / (P q_l) for a fast-BConv error u in [0, K + 1), i.e.
    # |R - C / (P q_l)| <= K + 1 -- checked against the big-integer division, not the RNS formula.
    n = 16
    qs, ps = _small_chain(n, 4)
    rng = random.Random(6)
    basis = qs + ps
    P = ps[0] * ps[1]
    for l in (3, 2, 1):
        qb = qs[: l + 1] + ps
        c = _rand_res(rng, qb, n)
        out = np.empty((l, n), dtype=np.uint64)
        orc.lib().or_moddown_rescale(n, l, orc._arr(qs), len(ps), orc._arr(ps), orc._arr(c), out)
        C, QP = big.crt([c[t] for t in range(len(qb))], qb)
        R, Q = big.crt([out[t] for t in range(l)], qs[:l])
        M = P * qs[l]
        for k in range(n):
            cc = big.centered(C[k], QP)
            rr = big.centered(R[k], Q)
            assert abs(rr * M - cc) <= (len(ps) + 2) * M
    del basis


def test_keyswitch_correctness_bound():
    # Dec_s(KS(x; s')) - x*s' is small, with keys made at the
    # top level and used at lower levels with truncated digits.
    P = toy(log_n=5, n_q=5, scale_bits=30, n_p=2, alpha=2)
    keys = orc.keygen(P, seed=9, rotations=[1])
    ev = orc.Evaluator(P, keys.rlk, keys.gk)
    basis = list(P.q) + list(P.p)
    rng = random.Random(1)
    s_res_full = orc.small_to_rns(keys.s, basis)
    s2_full = orc.poly_mul(basis, s_res_full, s_res_full)
    for l in (4, 3, 1):
        qs = list(P.q[: l + 1])
        x = _rand_res(rng, qs, P.n)
        d0, d1 = ev.keyswitch(x, l, keys.rlk)
        s = orc.small_to_rns(keys.s, qs)
        lhs = orc.poly_add(qs, d0, orc.poly_mul(qs, d1, s))
        rhs = orc.poly_mul(qs, x, s2_full[: l + 1])
        diff = orc.poly_sub(qs, lhs, rhs)
        D, Q = big.crt([diff[i] for i in range(l + 1)], qs)
        worst = max(abs(big.centered(v, Q)) for v in D)
        # |e_ks| <= dnum * N * B_e * max q_i / P + K-ish rounding: loose bound 2^20
        assert worst < (1 << 20), worst


def test_primes_rule():
    from synth.params import ps4
    P = ps4()
    assert all(is_prime(q) and (q - 1) % (2 * P.n) == 0 for q in P.q + P.p)
    assert len(set(P.q + P.p)) == len(P.q) + len(P.p)
    assert P.q[0] > max(P.p) and all(q < (1 << 60) for q in P.q + P.p)
