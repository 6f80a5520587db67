"""CKKS parameter sets PS1-PS4 and the pinned prime rule.

Prime rule (pinned; the paper only fixes bit sizes, Table
tab:ckks_params P:433-454, "Scaling mod. size 40/50 bits, First/last mod. size
60 bits"):
  * q0 and p_0..p_{K-1}: the largest primes = 1 (mod 2N) below 2^60, taken in
    descending order (q0 first);
  * scaling primes q1..qL: primes = 1 (mod 2N) alternating below and above
    2^Delta, nearest first.
Primes are parameters handed explicitly to both sides (the C-ABI takes them in
``mmfhe_params``); nothing here computes any CKKS arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases up to 41)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)
    for p in small:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def primes_below(bound: int, two_n: int, count: int, exclude=()) -> list[int]:
    """Largest `count` primes = 1 mod two_n strictly below `bound`, descending."""
    out = []
    c = ((bound - 2) // two_n) * two_n + 1
    while len(out) < count:
        if c >= bound:
            c -= two_n
            continue
        if c not in exclude and is_prime(c):
            out.append(c)
        c -= two_n
        if c < two_n:
            raise ValueError("ran out of primes")
    return out


def scaling_primes(bits: int, two_n: int, count: int, exclude=()) -> list[int]:
    """Primes = 1 mod two_n alternating below / above 2^bits, nearest first."""
    target = 1 << bits
    b = ((target - 1) // two_n) * two_n + 1
    if b >= target:
        b -= two_n
    a = b + two_n
    out: list[int] = []
    want_below = True
    while len(out) < count:
        if want_below:
            while not (is_prime(b) and b not in exclude and b not in out):
                b -= two_n
            out.append(b)
            b -= two_n
        else:
            while not (is_prime(a) and a not in exclude and a not in out):
                a += two_n
            out.append(a)
            a += two_n
        want_below = not want_below
    return out


@dataclass(frozen=True)
class ParamSet:
    name: str
    log_n: int
    q: tuple            # q_0 .. q_L
    p: tuple            # p_0 .. p_{K-1}
    alpha: int          # limbs per key-switching digit
    scale_bits: int
    note: str = ""

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def L(self) -> int:
        return len(self.q) - 1

    @property
    def K(self) -> int:
        return len(self.p)

    def dnum(self, level: int | None = None) -> int:
        lvl = self.L if level is None else level
        return -(-(lvl + 1) // self.alpha)


@lru_cache(maxsize=None)
def make_params(log_n: int, n_q: int, scale_bits: int, n_p: int, alpha: int,
                first_bits: int = 60, name: str = "custom") -> ParamSet:
    two_n = 2 << log_n
    big = primes_below(1 << first_bits, two_n, 1 + n_p)
    q0, ps = big[0], big[1:]
    qs = [q0] + scaling_primes(scale_bits, two_n, n_q - 1, exclude=set(big))
    return ParamSet(name, log_n, tuple(qs), tuple(ps), alpha, scale_bits)


def ps1() -> ParamSet:  # C1: N=2^13, Q=(60,40), P=(60), alpha=1
    return make_params(13, 2, 40, 1, 1, name="PS1")


def ps2() -> ParamSet:  # C2: N=2^14, Q=(60, 7x40), P=(60), alpha=1
    return make_params(14, 8, 40, 1, 1, name="PS2")


def ps3() -> ParamSet:  # C3: N=2^15, Q=(60, 11x50), P=4x60, alpha=4 (dnum 3)
    return make_params(15, 12, 50, 4, 4, name="PS3")


def ps4() -> ParamSet:  # C4/C5: N=2^16, Q=(60, 19x50), P=7x60, alpha=7 (dnum 3)
    return make_params(16, 20, 50, 7, 7, name="PS4")


def ps4d2() -> ParamSet:
    """PS4 with dnum 2 (SURVEY §8(d) lever 3): N=2^16, the same 20 Q limbs, alpha 10 and
    K = 10 special primes of 60 bits; log2 PQ ~ 1610 <= 1772 (128-bit, N = 2^16)."""
    return make_params(16, 20, 50, 10, 10, name="PS4d2")


def psv() -> ParamSet:
    """The paper's vital column: N=2^15, 11 Q limbs (60 + 10x40,
    the 5.5 MB ciphertext of P:1405), dnum 3 (the 22.5 MiB relinearisation key of P:1412:
    3 digits x 2 x 15 limbs x 2^15 x 8 B): alpha 4, K = 4 special primes of 60 bits;
    log2 PQ ~ 700 <= 881 (128-bit, ternary, N = 2^15)."""
    return make_params(15, 11, 40, 4, 4, name="PSV")


def toy(log_n: int = 10, n_q: int = 6, scale_bits: int = 40, n_p: int = 2,
        alpha: int = 2) -> ParamSet:
    """Small, insecure sets for fast tests (same prime rule)."""
    return make_params(log_n, n_q, scale_bits, n_p, alpha, name=f"toy{log_n}")


PARAM_SETS = {"PS1": ps1, "PS2": ps2, "PS3": ps3, "PS4": ps4, "PS4d2": ps4d2, "PSV": psv}
