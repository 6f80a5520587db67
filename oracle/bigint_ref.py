"""O-BIG: tiny-N, non-RNS ring arithmetic with Python big integers --
TEST INFRASTRUCTURE ONLY.

It is the independent model O-RNS (``ckks_ref.c``) is pinned against
(SURVEY §8(c)-9): the ring Z_Q[X]/(X^N+1) of PAPER.md P:391 written out with
schoolbook negacyclic products, the CRT, and the round-half-up division that
the pinned rescale must equal.  Pure-Python loops: only for
N <= 64.
"""
from __future__ import annotations


def schoolbook_negacyclic(a, b, q: int | None = None):
    """c = a*b mod (X^N + 1): c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j."""
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k < n:
                c[k] += a[i] * b[j]
            else:
                c[k - n] -= a[i] * b[j]
    if q is not None:
        c = [x % q for x in c]
    return c


def crt(residues, qs):
    """The unique X in [0, prod qs) with X = r_i mod q_i (per coefficient)."""
    Q = 1
    for q in qs:
        Q *= q
    n = len(residues[0])
    out = []
    for k in range(n):
        x = 0
        for r, q in zip(residues, qs):
            qh = Q // q
            x += (int(r[k]) * pow(qh, -1, q) % q) * qh
        out.append(x % Q)
    return out, Q


def centered(x: int, Q: int) -> int:
    x %= Q
    return x - Q if x > Q // 2 else x


def round_half_up_div(a: int, d: int) -> int:
    """round(a/d) with ties toward +infinity: floor((a + floor(d/2)) / d) for odd d."""
    return (a + d // 2) // d


def galois_apply(a, g: int):
    """a(X) -> a(X^g) on integer coefficients (negacyclic wrap)."""
    n = len(a)
    out = [0] * n
    for i, x in enumerate(a):
        j = (i * g) % (2 * n)
        if j < n:
            out[j] += x
        else:
            out[j - n] -= x
    return out
