"""Counter-based SplitMix64 streams and the RLWE samplers built on them.

SURVEY §8(d) "PRNG": keys and encryption use a counter-based, platform
independent generator keyed by (seed, stream id).  Draw i of stream (seed, sid)
is mix64(key(seed, sid) + (i+1)*GOLDEN) -- a pure function of its index, so any
slice of a stream can be regenerated independently.

Samplers (the paper is silent on the distributions, PAPER.md P:694 only names
the keys; readings in DESIGN.md §3):
  * uniform residues mod q: floor(x*q / 2^64) (multiply-shift, bias < q/2^64);
  * ternary secret: x mod 3 - 1;
  * error: centered binomial CBD(eta=21), variance 10.5 (sigma 3.24 ~ the
    HE-standard 3.2 that SPEC S:147 names), integer-only so it is bit-stable.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_M32 = np.uint64(0xFFFFFFFF)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, sid: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = mix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))
        k = mix64(k ^ np.array([sid & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))
    return k[0]


def draws(seed: int, sid: int, n: int, offset: int = 0) -> np.ndarray:
    """n raw 64-bit draws of stream (seed, sid) starting at index offset."""
    key = stream_key(seed, sid)
    i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(key + i * GOLDEN)


def mulhi64(x: np.ndarray, q: int) -> np.ndarray:
    """floor(x*q / 2^64) for uint64 arrays x and scalar q < 2^64."""
    x = np.asarray(x, dtype=np.uint64)
    qh, ql = np.uint64(q >> 32), np.uint64(q & 0xFFFFFFFF)
    xh, xl = x >> np.uint64(32), x & _M32
    with np.errstate(over="ignore"):
        ll = xl * ql
        lh = xl * qh
        hl = xh * ql
        hh = xh * qh
        mid = (ll >> np.uint64(32)) + (lh & _M32) + (hl & _M32)
        return hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))


def uniform_mod(seed: int, sid: int, n: int, q: int, offset: int = 0) -> np.ndarray:
    """n residues in [0, q) (uint64) from draws offset..offset+n-1."""
    return mulhi64(draws(seed, sid, n, offset), q)


def ternary(seed: int, sid: int, n: int) -> np.ndarray:
    """n values in {-1, 0, 1} (int64)."""
    return (draws(seed, sid, n) % np.uint64(3)).astype(np.int64) - 1


def cbd(seed: int, sid: int, n: int, eta: int = 21) -> np.ndarray:
    """Centered binomial: popcount(eta bits) - popcount(next eta bits), int64."""
    assert 2 * eta <= 64
    x = draws(seed, sid, n)
    m = np.uint64((1 << eta) - 1)
    a = np.bitwise_count(x & m).astype(np.int64)
    b = np.bitwise_count((x >> np.uint64(eta)) & m).astype(np.int64)
    return a - b


# stream ids: one per purpose so that draws never overlap
SID_SECRET = 1
SID_PK_A = 2
SID_PK_E = 3
SID_KS_A = 1 << 32        # + 64*key_index + digit   (limb t at offset t*N)
SID_KS_E = 2 << 32        # + 64*key_index + digit
SID_ENC_U = 3 << 32       # + 4*ct_index
SID_ENC_E0 = (3 << 32) + 1
SID_ENC_E1 = (3 << 32) + 2
SID_UNIFORM = 4 << 32     # bench: uniform residues standing in for ciphertexts/keys
