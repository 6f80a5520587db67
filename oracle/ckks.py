"""O-RNS: plain RNS-CKKS on the CPU -- TEST INFRASTRUCTURE ONLY.

Client side (keygen, encode, encrypt, decrypt) and the cloud evaluator ops the
mmFHE kernels are built from.  Ciphertext polynomials are kept in COEFFICIENT
form as uint64 arrays [n_limbs][N]; every ring product goes through the
textbook NTT of ``ckks_ref.c``.  Parity is pinned only where SURVEY §8(c)
pins it: exact ring operations (c-4) and the pinned non-exact steps (c-5),
with the scale/level rules of c-6.

Paper passages:
  * ring Z_Q[X]/(X^N+1), ciphertext = pair of polynomials
  * KeyGen -> sk, pk, rlk, gk; one Galois key per rotation k
  * N/2 real slots, slot-wise add/mult, rotation
  * Addition free, multiplication consumes a level, Rot(Enc(a),k) P:416-421
  * re and im are encrypted as separate ciphertexts
Readings where the paper is silent: canonical embedding
slot j <-> zeta^(5^j mod 2N); left rotation Rot(v,k)[j] = v[(j+k) mod n];
Galois element g = 5^(k mod N/2) mod 2N; ternary secret; CBD(21) errors.
Complex slots (reading R28): the same embedding carries a complex
vector z (coefficients stay real: m(zeta^-e) = conj m(zeta^e)); the conjugation
automorphism X -> X^(2N-1) conjugates every slot and has its own key (id CONJ).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from synth import prng
from synth.params import ParamSet

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libckks_ref.so")
_lib = None

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile ckks_ref.c (plain C, -O2, OpenMP across independent limbs) into
    oracle/_build/libckks_ref.so."""
    src = os.path.join(_HERE, "ckks_ref.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-shared", "-fPIC", src, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        _lib.or_find_psi.restype = u64
        _lib.or_find_psi.argtypes = [u64, u32]
        _lib.or_ntt_forward.argtypes = [u32, u64, u64p]
        _lib.or_ntt_inverse.argtypes = [u32, u64, u64p]
        _lib.or_poly_mul.argtypes = [u32, u32, u64p, u64p, u64p, u64p]
        for f in (_lib.or_add, _lib.or_sub, _lib.or_scalar_mul):
            f.argtypes = [u32, u32, u64p, u64p, u64p, u64p]
            f.restype = None
        _lib.or_automorphism.argtypes = [u32, u32, u64p, u64p, u64, u64p]
        _lib.or_automorphism.restype = None
        _lib.or_rescale.argtypes = [u32, u32, u64p, u64p, u64p]
        _lib.or_rescale.restype = None
        _lib.or_modup.argtypes = [u32, u32, u64p, u32, u64p, u32, u32, u64p, u64p]
        _lib.or_modup.restype = None
        _lib.or_moddown.argtypes = [u32, u32, u64p, u32, u64p, u64p, u64p]
        _lib.or_moddown.restype = None
        _lib.or_moddown_rescale.argtypes = [u32, u32, u64p, u32, u64p, u64p, u64p]
        _lib.or_moddown_rescale.restype = None
        _lib.or_keyswitch.argtypes = [u32, u32, u32, u64p, u32, u64p, u32, u64p, u64p, u64p, u64p]
    return _lib


def _arr(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.uint64)


# --------------------------------------------------------------------------
# ring helpers (coefficient form, limb-major)
# --------------------------------------------------------------------------

def poly_mul(qs, a, b):
    qs, a, b = _arr(qs), _arr(a), _arr(b)
    out = np.empty_like(a)
    rc = lib().or_poly_mul(a.shape[-1], len(qs), qs, a, b, out)
    assert rc == 0, "prime not NTT-friendly"
    return out


def poly_add(qs, a, b):
    qs, a, b = _arr(qs), _arr(a), _arr(b)
    out = np.empty_like(a)
    lib().or_add(a.shape[-1], len(qs), qs, a, b, out)
    return out


def poly_sub(qs, a, b):
    qs, a, b = _arr(qs), _arr(a), _arr(b)
    out = np.empty_like(a)
    lib().or_sub(a.shape[-1], len(qs), qs, a, b, out)
    return out


def poly_scalar(qs, a, c):
    qs, a, c = _arr(qs), _arr(a), _arr(c)
    out = np.empty_like(a)
    lib().or_scalar_mul(a.shape[-1], len(qs), qs, a, c, out)
    return out


def automorphism(qs, a, g):
    qs, a = _arr(qs), _arr(a)
    out = np.empty_like(a)
    lib().or_automorphism(a.shape[-1], len(qs), qs, a, int(g), out)
    return out


def small_to_rns(v: np.ndarray, qs) -> np.ndarray:
    """Signed int64 (small) coefficients -> residues [len(qs)][N]."""
    v = np.asarray(v, dtype=np.int64)
    return np.stack([np.mod(v, np.int64(q)).astype(np.uint64) for q in qs])


def bigint_to_rns(v, qs) -> np.ndarray:
    """Python-int coefficients (object array) -> residues."""
    v = np.asarray(v, dtype=object)
    return np.stack([np.array([int(x) % q for x in v], dtype=np.uint64) for q in qs])


def crt_centered(res: np.ndarray, qs) -> np.ndarray:
    """CRT-reconstruct residues [l+1][N] to integers in (-Q/2, Q/2] (object array)."""
    qs = [int(q) for q in qs]
    Q = 1
    for q in qs:
        Q *= q
    acc = np.zeros(res.shape[-1], dtype=object)
    for i, q in enumerate(qs):
        qhat = Q // q
        inv = pow(qhat % q, -1, q)
        t = [(int(x) * inv) % q for x in res[i]]
        acc = acc + np.array(t, dtype=object) * qhat
    acc = acc % Q
    half = Q // 2
    return np.where(acc > half, acc - Q, acc)


# --------------------------------------------------------------------------
# canonical embedding: slot j <-> zeta^(5^j mod 2N), zeta = e^(i pi/N)
# --------------------------------------------------------------------------

def _slot_positions(n_ring: int):
    two_n = 2 * n_ring
    e = np.empty(n_ring // 2, dtype=np.int64)
    x = 1
    for j in range(n_ring // 2):
        e[j] = x
        x = x * 5 % two_n
    pos = (e - 1) // 2                  # index k of root zeta^(2k+1)
    pos_conj = (two_n - e - 1) // 2     # conjugate root zeta^(-5^j)
    return pos, pos_conj


def embed_inverse(z: np.ndarray, n_ring: int) -> np.ndarray:
    """Real coefficients m with m(zeta^(5^j)) = z_j for all N/2 slots.
    m(zeta^(2k+1)) = sum_i (m_i zeta^i) omega^(ik), omega = zeta^2, so
    m_i zeta^i = fft(E)_i / N and m_i = that * zeta^(-i)."""
    pos, pos_conj = _slot_positions(n_ring)
    E = np.zeros(n_ring, dtype=np.complex128)
    E[pos] = z
    E[pos_conj] = np.conj(z)
    i = np.arange(n_ring)
    b = np.fft.fft(E) / n_ring
    return (b * np.exp(-1j * np.pi * i / n_ring)).real


def embed(m: np.ndarray, n_ring: int) -> np.ndarray:
    """Slot values z_j = m(zeta^(5^j)) of real coefficients m."""
    pos, _ = _slot_positions(n_ring)
    i = np.arange(n_ring)
    b = np.asarray(m, dtype=np.float64) * np.exp(1j * np.pi * i / n_ring)
    E = np.fft.ifft(b) * n_ring
    return E[pos]


def replicate(v: np.ndarray, n_ring: int) -> np.ndarray:
    """Sparse packing: period-n vector replicated N/(2n) times (real, or
    complex slot values, reading R28)."""
    v = np.asarray(v)
    v = v.astype(np.complex128) if np.iscomplexobj(v) else v.astype(np.float64)
    n = len(v)
    assert (n_ring // 2) % n == 0, "packing period must divide N/2"
    return np.tile(v, (n_ring // 2) // n)


def encode(P: ParamSet, v, scale: float, level: int) -> np.ndarray:
    """round(scale * embed^-1(replicate(v))) as residues mod q_0..q_level."""
    m = embed_inverse(replicate(v, P.n), P.n) * float(scale)
    m = np.rint(m)
    assert np.max(np.abs(m)) < 2.0 ** 62, "encoding overflow"
    mi = m.astype(np.int64)
    return small_to_rns(mi, P.q[: level + 1])


def encode_pq(P: ParamSet, v, scale: float, level: int) -> np.ndarray:
    """The same integer encoding as encode(), reduced mod q_0..q_level, p_0..p_{K-1}: the
    form in which double-hoisted BSGS multiplies its diagonals."""
    m = np.rint(embed_inverse(replicate(v, P.n), P.n) * float(scale))
    assert np.max(np.abs(m)) < 2.0 ** 62, "encoding overflow"
    return small_to_rns(m.astype(np.int64), list(P.q[: level + 1]) + list(P.p))


def decode(P: ParamSet, res: np.ndarray, level: int, scale: float, n_slots: int,
           complex_out: bool = False) -> np.ndarray:
    """Slot values of a plaintext (real parts, or complex with complex_out, reading R28)."""
    ints = crt_centered(res, P.q[: level + 1])
    m = np.array([float(x) for x in ints]) / float(scale)
    z = embed(m, P.n)[:n_slots]
    return z if complex_out else z.real


def encode_scalar(c: float, q_l: int) -> int:
    """Exact round-half-away(c * q_l) (SURVEY §8(c)-5 scalar-constant encoding)."""
    x = Fraction(c) * q_l
    s = -1 if x < 0 else 1
    return s * int(abs(x) + Fraction(1, 2))


# --------------------------------------------------------------------------
# keys -- SecretKey never leaves the client; the cloud gets pk, rlk, gk
# --------------------------------------------------------------------------

@dataclass
class Keys:
    s: np.ndarray                        # int64 ternary coefficients
    pk: tuple                            # (b, a) over q_0..q_L
    rlk: np.ndarray | None = None        # [dnum][2][L+1+K][N]
    gk: dict = field(default_factory=dict)  # k (normalised) -> [dnum][2][L+1+K][N]


# Key id of the conjugation automorphism (reading R28): outside every normalised rotation
# amount [0, N/2); the C ABI uses the same value (MMFHE_STEP_CONJ = INT32_MIN).
CONJ = -(1 << 31)
# Key id of the conjugate-product key (reading R32): the key switching s * sigma_{2N-1}(s) to s, which
# relinearises a product d * sigma_{2N-1}(d) directly (C ABI: MMFHE_STEP_CONJ_PROD = INT32_MIN + 1).
CONJ_PROD = CONJ + 1


def galois_element(P: ParamSet, k: int) -> int:
    """g = 5^(k mod N/2) mod 2N; k is normalised to [0, N/2) first.
    k = CONJ: g = 2N - 1 = -1 mod 2N, the complex conjugation of every slot (reading R28:
    zeta^(5^j) -> zeta^(-5^j) = conj zeta^(5^j))."""
    if k == CONJ:
        return 2 * P.n - 1
    return pow(5, k % (P.n // 2), 2 * P.n)


def key_id(P: ParamSet, k: int) -> int:
    """Normalised Galois-key id: k mod N/2 for a rotation, CONJ / CONJ_PROD for the conjugation and
    the conjugate-product key."""
    return k if k in (CONJ, CONJ_PROD) else k % (P.n // 2)


def key_index(P: ParamSet, kid: int) -> int:
    """PRNG stream index of a key (make_evk): 1 + k for rotation k in [1, N/2), 1 + N/2 for the
    conjugation, 2 + N/2 for the conjugate-product key (0 is the relinearisation key)."""
    if kid == CONJ:
        return 1 + P.n // 2
    if kid == CONJ_PROD:
        return 2 + P.n // 2
    return 1 + kid


def _full_basis(P: ParamSet):
    return list(P.q) + list(P.p)


def make_evk(P: ParamSet, s: np.ndarray, s_prime_res: np.ndarray, seed: int, key_index: int) -> np.ndarray:
    """evk_j = (b_j, a_j) over P*Q_L, b_j = -a_j s + e_j + P g_j s' with
    g_j = 1 mod q_i for i in I_j (full digit at level L), 0 for other q_i
    (SURVEY §8(c)-5 "Keys").  s_prime_res: residues of s' over the full basis."""
    basis = _full_basis(P)
    nb = len(basis)
    L = P.L
    dnum = P.dnum()
    s_res = small_to_rns(s, basis)
    Pmod = [1] * nb
    for i, q in enumerate(basis):
        prod = 1
        for p in P.p:
            prod = prod * p % q
        Pmod[i] = prod
    out = np.empty((dnum, 2, nb, P.n), dtype=np.uint64)
    for j in range(dnum):
        a = np.stack([prng.uniform_mod(seed, prng.SID_KS_A + 64 * key_index + j, P.n, q, offset=t * P.n)
                      for t, q in enumerate(basis)])
        e = small_to_rns(prng.cbd(seed, prng.SID_KS_E + 64 * key_index + j, P.n), basis)
        b = poly_sub(basis, e, poly_mul(basis, a, s_res))
        lo, hi = j * P.alpha, min(j * P.alpha + P.alpha, L + 1)
        gadget = np.zeros(nb, dtype=np.uint64)
        for i in range(lo, hi):
            gadget[i] = Pmod[i]
        b = poly_add(basis, b, poly_scalar(basis, s_prime_res, gadget))
        out[j, 0] = b
        out[j, 1] = a
    return out


def keygen(P: ParamSet, seed: int, rotations=(), relin: bool = True) -> Keys:
    basis = _full_basis(P)
    s = prng.ternary(seed, prng.SID_SECRET, P.n)
    qs = list(P.q)
    a = np.stack([prng.uniform_mod(seed, prng.SID_PK_A, P.n, q, offset=t * P.n) for t, q in enumerate(qs)])
    e = small_to_rns(prng.cbd(seed, prng.SID_PK_E, P.n), qs)
    b = poly_sub(qs, e, poly_mul(qs, a, small_to_rns(s, qs)))
    keys = Keys(s=s, pk=(b, a))
    s_res = small_to_rns(s, basis)
    if relin:
        keys.rlk = make_evk(P, s, poly_mul(basis, s_res, s_res), seed, 0)
    for k in sorted({key_id(P, r) for r in rotations} - {0}):
        if k == CONJ_PROD:  # s * sigma_{2N-1}(s) (reading R32)
            sp = poly_mul(basis, s_res, automorphism(basis, s_res, 2 * P.n - 1))
            keys.gk[k] = make_evk(P, s, sp, seed, key_index(P, k))
            continue
        g = galois_element(P, k)
        keys.gk[k] = make_evk(P, s, automorphism(basis, s_res, g), seed, key_index(P, k))
    return keys


# --------------------------------------------------------------------------
# ciphertexts
# --------------------------------------------------------------------------

@dataclass
class Ct:
    c: list            # polys, each uint64 [level+1][N]; 2 (or 3 after a tensor)
    level: int
    scale: float
    n_slots: int

    def copy(self) -> "Ct":
        return Ct([x.copy() for x in self.c], self.level, self.scale, self.n_slots)


def encrypt(P: ParamSet, keys: Keys, pt: np.ndarray, level: int, scale: float, n_slots: int,
            seed: int, index: int) -> Ct:
    """pk-encryption at `level`: c0 = u*b + e0 + m, c1 = u*a + e1 (the pk
    limbs q_{level+1..L} are dropped)."""
    qs = list(P.q[: level + 1])
    b, a = keys.pk[0][: level + 1], keys.pk[1][: level + 1]
    u = small_to_rns(prng.ternary(seed, prng.SID_ENC_U + 4 * index, P.n), qs)
    e0 = small_to_rns(prng.cbd(seed, prng.SID_ENC_E0 + 4 * index, P.n), qs)
    e1 = small_to_rns(prng.cbd(seed, prng.SID_ENC_E1 + 4 * index, P.n), qs)
    c0 = poly_add(qs, poly_add(qs, poly_mul(qs, u, b), e0), pt)
    c1 = poly_add(qs, poly_mul(qs, u, a), e1)
    return Ct([c0, c1], level, float(scale), n_slots)


def encrypt_vector(P, keys, v, level, seed, index, scale=None) -> Ct:
    scale = float(2 ** P.scale_bits) if scale is None else scale
    return encrypt(P, keys, encode(P, v, scale, level), level, scale, len(v), seed, index)


def decrypt(P: ParamSet, keys: Keys, ct: Ct) -> np.ndarray:
    """Residues of c0 + c1*s (+ c2*s^2) mod q_0..q_level."""
    qs = list(P.q[: ct.level + 1])
    s = small_to_rns(keys.s, qs)
    m = poly_add(qs, ct.c[0], poly_mul(qs, ct.c[1], s))
    if len(ct.c) == 3:
        m = poly_add(qs, m, poly_mul(qs, ct.c[2], poly_mul(qs, s, s)))
    return m


def decrypt_vector(P, keys, ct: Ct, complex_out: bool = False) -> np.ndarray:
    return decode(P, decrypt(P, keys, ct), ct.level, ct.scale, ct.n_slots, complex_out)


# --------------------------------------------------------------------------
# evaluator (cloud side)
# --------------------------------------------------------------------------

class DepthError(Exception):
    pass


class ScaleError(Exception):
    pass


class Evaluator:
    """Cloud-side ops with the pinned semantics of SURVEY §8(c)-4..6.
    `trace` records (op, level, arg) per call -- data-independent by
    construction (Theorem P:999-1006)."""

    def __init__(self, P: ParamSet, rlk=None, gk=None):
        self.P = P
        self.rlk = rlk
        self.gk = gk or {}
        self.trace: list = []

    # --- helpers
    def qs(self, level):
        return list(self.P.q[: level + 1])

    def _rec(self, op, level, arg=""):
        self.trace.append((op, level, arg))

    # --- exact ops (c-4)
    def add(self, a: Ct, b: Ct) -> Ct:
        self._check_pair(a, b)
        self._rec("hadd", a.level)
        qs = self.qs(a.level)
        return Ct([poly_add(qs, x, y) for x, y in zip(a.c, b.c)], a.level, a.scale, a.n_slots)

    def sub(self, a: Ct, b: Ct) -> Ct:
        self._check_pair(a, b)
        self._rec("hsub", a.level)
        qs = self.qs(a.level)
        return Ct([poly_sub(qs, x, y) for x, y in zip(a.c, b.c)], a.level, a.scale, a.n_slots)

    def _check_pair(self, a: Ct, b: Ct):
        if a.level != b.level or len(a.c) != len(b.c):
            raise ValueError("level/size mismatch")
        if a.scale != b.scale:
            raise ScaleError(f"scale mismatch {a.scale} vs {b.scale}")

    def drop_to(self, a: Ct, level: int) -> Ct:
        """Mod-switch by dropping limbs q_{level+1..} (exact, scale unchanged)."""
        if level > a.level:
            raise ValueError("cannot raise level")
        if level == a.level:
            return a
        self._rec("modswitch", a.level, str(level))
        return Ct([x[: level + 1].copy() for x in a.c], level, a.scale, a.n_slots)

    def pmult(self, a: Ct, pt: np.ndarray, pt_scale: float) -> Ct:
        """Vector-plaintext product; pt are residues [level+1][N] at the ct's level."""
        self._rec("pmult", a.level)
        qs = self.qs(a.level)
        return Ct([poly_mul(qs, x, pt[: a.level + 1]) for x in a.c], a.level, a.scale * pt_scale, a.n_slots)

    def pmult_scalar(self, a: Ct, c: float) -> Ct:
        """Scalar constant encoded at Delta_pt = q_level (c-5 exact rounding)."""
        self._rec("pmult_scalar", a.level)
        qs = self.qs(a.level)
        ql = self.P.q[a.level]
        v = encode_scalar(c, ql)
        res = np.array([v % q for q in qs], dtype=np.uint64)
        return Ct([poly_scalar(qs, x, res) for x in a.c], a.level, a.scale * ql, a.n_slots)

    def tensor(self, a: Ct, b: Ct) -> Ct:
        """(a0 b0, a0 b1 + a1 b0, a1 b1); scale s_a s_b (c-4, c-6)."""
        if a.level != b.level:
            raise ValueError("level mismatch")
        self._rec("tensor", a.level)
        qs = self.qs(a.level)
        d0 = poly_mul(qs, a.c[0], b.c[0])
        d1 = poly_add(qs, poly_mul(qs, a.c[0], b.c[1]), poly_mul(qs, a.c[1], b.c[0]))
        d2 = poly_mul(qs, a.c[1], b.c[1])
        return Ct([d0, d1, d2], a.level, a.scale * b.scale, a.n_slots)

    # --- key switching (c-5)
    def keyswitch(self, x: np.ndarray, level: int, evk: np.ndarray):
        P = self.P
        d0 = np.empty((level + 1, P.n), dtype=np.uint64)
        d1 = np.empty_like(d0)
        rc = lib().or_keyswitch(P.n, level, P.L, _arr(P.q), P.K, _arr(P.p), P.alpha,
                                _arr(x), _arr(evk), d0, d1)
        assert rc == 0
        return d0, d1

    def relin(self, a: Ct) -> Ct:
        """(c0 + d0, c1 + d1), (d0, d1) = KS(c2; rlk)."""
        if len(a.c) != 3:
            raise ValueError("relin needs a 3-poly ciphertext")
        if self.rlk is None:
            raise KeyError("missing relinearisation key")
        self._rec("relin", a.level)
        qs = self.qs(a.level)
        d0, d1 = self.keyswitch(a.c[2], a.level, self.rlk)
        return Ct([poly_add(qs, a.c[0], d0), poly_add(qs, a.c[1], d1)], a.level, a.scale, a.n_slots)

    def rotate(self, a: Ct, k: int) -> Ct:
        """HRot: (sigma_g c0 + d0, d1), (d0, d1) = KS(sigma_g c1; gk_k);
        automorphism first (c-5).  Rot(v,k)[j] = v[(j+k) mod n]."""
        P = self.P
        kn = k % (P.n // 2)
        if kn == 0:
            return a
        if kn not in self.gk:
            raise KeyError(f"missing Galois key for rotation {kn}")
        self._rec("hrot", a.level, str(kn))
        return self._automorphism_ks(a, galois_element(P, kn), self.gk[kn])

    def _automorphism_ks(self, a: Ct, g: int, evk: np.ndarray) -> Ct:
        qs = self.qs(a.level)
        c0 = automorphism(qs, a.c[0], g)
        c1 = automorphism(qs, a.c[1], g)
        d0, d1 = self.keyswitch(c1, a.level, evk)
        return Ct([poly_add(qs, c0, d0), d1], a.level, a.scale, a.n_slots)

    def conjugate(self, a: Ct) -> Ct:
        """Conj (reading R28): (sigma_g c0 + d0, d1), (d0, d1) = KS(sigma_g c1; gk_CONJ) with
        g = 2N - 1 -- HRot's algorithm with the conjugation's Galois element; every slot
        value is conjugated."""
        if CONJ not in self.gk:
            raise KeyError("missing conjugation key")
        self._rec("conj", a.level)
        return self._automorphism_ks(a, galois_element(self.P, CONJ), self.gk[CONJ])

    def rotate_hoisted(self, a: Ct, ks) -> list:
        """Hoisted HRot (a separate op): ModUp(c1) once, then per step
        (sigma_g c0 + d0, d1) with (d0, d1) = ModDown(sum_j sigma_g(y_j) (.) evk_g,j).
        sigma_g acts on the ModUp'd digits over Q_l u P, so residues differ from
        rotate() (BConv does not commute with sigma_g's sign flips)."""
        ys = self.hoist_modup(a)
        return [self.hoisted_step(a, ys, k) for k in ks]

    def hoist_modup(self, a: Ct) -> list:
        """ModUp of every digit of c1 (coefficient form over Q_l u P), shared by the
        hoisted rotations of `a`."""
        P = self.P
        l = a.level
        ys = []
        for j in range(-(-(l + 1) // P.alpha)):
            y = np.empty((l + 1 + P.K, P.n), dtype=np.uint64)
            lib().or_modup(P.n, l, _arr(P.q), P.K, _arr(P.p), P.alpha, j, _arr(a.c[1]), y)
            ys.append(y)
        return ys

    def hoisted_step(self, a: Ct, ys: list, k: int) -> Ct:
        P = self.P
        l = a.level
        kn = k % (P.n // 2)
        if kn == 0:
            return a
        if kn not in self.gk:
            raise KeyError(f"missing Galois key for rotation {kn}")
        self._rec("hrot_hoisted", l, str(kn))
        basis = list(P.q[: l + 1]) + list(P.p)
        nkey = P.L + 1 + P.K
        g = galois_element(P, kn)
        evk = self.gk[kn]
        acc0 = np.zeros((l + 1 + P.K, P.n), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for j, y in enumerate(ys):
            sy = automorphism(basis, y, g)
            kb = np.concatenate([evk[j, 0, : l + 1], evk[j, 0, P.L + 1: nkey]])
            ka = np.concatenate([evk[j, 1, : l + 1], evk[j, 1, P.L + 1: nkey]])
            acc0 = poly_add(basis, acc0, poly_mul(basis, sy, kb))
            acc1 = poly_add(basis, acc1, poly_mul(basis, sy, ka))
        d0 = np.empty((l + 1, P.n), dtype=np.uint64)
        d1 = np.empty_like(d0)
        lib().or_moddown(P.n, l, _arr(P.q), P.K, _arr(P.p), _arr(acc0), d0)
        lib().or_moddown(P.n, l, _arr(P.q), P.K, _arr(P.p), _arr(acc1), d1)
        qs = self.qs(l)
        return Ct([poly_add(qs, automorphism(qs, a.c[0], g), d0), d1], l, a.scale, a.n_slots)

    # --- double hoisting ("baby steps in PQ with P sigma(c0) lift,
    # diagonals encoded in PQ, one ModDown per giant group" -- a third op, pinned here).
    # A PQ ciphertext holds P * (a ciphertext) over the extended basis Q_l u P: rows
    # q_0..q_l then p_0..p_{K-1} per polynomial (level = l).
    def pq_basis(self, level):
        return list(self.P.q[: level + 1]) + list(self.P.p)

    def _p_mod(self, basis):
        Pm = 1
        for p in self.P.p:
            Pm *= int(p)
        return np.array([Pm % int(t) for t in basis], dtype=np.uint64)

    def lift_pq(self, a: Ct) -> Ct:
        """(P c0, P c1) over Q_l u P (zero mod every p_k): the identity baby step."""
        self._rec("lift_pq", a.level)
        basis = self.pq_basis(a.level)
        pm = self._p_mod(basis)
        l1 = a.level + 1
        out = []
        for x in a.c:
            y = np.zeros((len(basis), self.P.n), dtype=np.uint64)
            y[:l1] = poly_scalar(basis[:l1], x, pm[:l1])
            out.append(y)
        return Ct(out, a.level, a.scale, a.n_slots)

    def hoisted_step_pq(self, a: Ct, ys: list, k: int) -> Ct:
        """A hoisted rotation left in PQ: (P sigma_g(c0) + sum_j sigma_g(y_j) (.) b_j,
        sum_j sigma_g(y_j) (.) a_j) over Q_l u P -- the hoisted HRot without its ModDown."""
        P = self.P
        l = a.level
        kn = k % (P.n // 2)
        if kn == 0:
            return self.lift_pq(a)
        if kn not in self.gk:
            raise KeyError(f"missing Galois key for rotation {kn}")
        self._rec("hrot_hoisted_pq", l, str(kn))
        basis = self.pq_basis(l)
        nkey = P.L + 1 + P.K
        g = galois_element(P, kn)
        evk = self.gk[kn]
        acc0 = np.zeros((l + 1 + P.K, P.n), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for j, y in enumerate(ys):
            sy = automorphism(basis, y, g)
            kb = np.concatenate([evk[j, 0, : l + 1], evk[j, 0, P.L + 1: nkey]])
            ka = np.concatenate([evk[j, 1, : l + 1], evk[j, 1, P.L + 1: nkey]])
            acc0 = poly_add(basis, acc0, poly_mul(basis, sy, kb))
            acc1 = poly_add(basis, acc1, poly_mul(basis, sy, ka))
        pm = self._p_mod(basis)
        c0 = np.zeros_like(acc0)
        c0[: l + 1] = poly_scalar(basis[: l + 1], automorphism(self.qs(l), a.c[0], g), pm[: l + 1])
        return Ct([poly_add(basis, acc0, c0), acc1], l, a.scale, a.n_slots)

    def moddown_poly(self, x: np.ndarray, level: int) -> np.ndarray:
        """ModDown of one polynomial over Q_l u P to Q_l."""
        P = self.P
        out = np.empty((level + 1, P.n), dtype=np.uint64)
        lib().or_moddown(P.n, level, _arr(P.q), P.K, _arr(P.p), _arr(x), out)
        return out

    def rotate_pq(self, a: Ct, k: int) -> Ct:
        """Giant step of double-hoisted BSGS on a PQ ciphertext a = (a0, a1):
        a1' = ModDown(a1) (to Q_l), then the rotation's key switch without ModDown:
        (sigma_g(a0) + sum_j y_j (.) b_j, sum_j y_j (.) a_j) over Q_l u P with
        y_j = ModUp_j(sigma_g(a1')) -- ModDown first, then the automorphism (BConv does not
        commute with sigma_g's sign flips, so the order is pinned)."""
        P = self.P
        l = a.level
        kn = k % (P.n // 2)
        if kn == 0:
            return a
        if kn not in self.gk:
            raise KeyError(f"missing Galois key for rotation {kn}")
        self._rec("hrot_pq", l, str(kn))
        basis = self.pq_basis(l)
        nkey = P.L + 1 + P.K
        g = galois_element(P, kn)
        evk = self.gk[kn]
        x = automorphism(self.qs(l), self.moddown_poly(a.c[1], l), g)
        acc0 = np.zeros((l + 1 + P.K, P.n), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for j in range(-(-(l + 1) // P.alpha)):
            y = np.empty((l + 1 + P.K, P.n), dtype=np.uint64)
            lib().or_modup(P.n, l, _arr(P.q), P.K, _arr(P.p), P.alpha, j, _arr(x), y)
            kb = np.concatenate([evk[j, 0, : l + 1], evk[j, 0, P.L + 1: nkey]])
            ka = np.concatenate([evk[j, 1, : l + 1], evk[j, 1, P.L + 1: nkey]])
            acc0 = poly_add(basis, acc0, poly_mul(basis, y, kb))
            acc1 = poly_add(basis, acc1, poly_mul(basis, y, ka))
        return Ct([poly_add(basis, automorphism(basis, a.c[0], g), acc0), acc1], l, a.scale, a.n_slots)

    def add_pq(self, a: Ct, b: Ct) -> Ct:
        self._check_pair(a, b)
        self._rec("hadd_pq", a.level)
        basis = self.pq_basis(a.level)
        return Ct([poly_add(basis, x, y) for x, y in zip(a.c, b.c)], a.level, a.scale, a.n_slots)

    def moddown_rescale_poly(self, x: np.ndarray, level: int) -> np.ndarray:
        """ModDown and rescale as one division by P q_level (reading R31) of one polynomial over
        Q_l u P: BConv of its p_0..p_{K-1}, q_l residues to q_0..q_{l-1}, out = (x - w) (P q_l)^{-1}."""
        P = self.P
        out = np.empty((level, P.n), dtype=np.uint64)
        lib().or_moddown_rescale(P.n, level, _arr(P.q), P.K, _arr(P.p), _arr(x), out)
        return out

    def moddown_rescale_ct(self, a: Ct) -> Ct:
        """A PQ ciphertext brought down to Q_{l-1} in one division (ModDown, then rescale, merged:
        reading R31); scale / q_l."""
        if a.level == 0:
            raise DepthError("depth exhausted")
        self._rec("moddown_rescale", a.level)
        return Ct([self.moddown_rescale_poly(x, a.level) for x in a.c], a.level - 1, a.scale / self.P.q[a.level],
                  a.n_slots)

    def relin_rescale_merged(self, a: Ct) -> Ct:
        """Relinearisation and rescale with one division (reading R31): the inner product of
        ModUp(c2) with rlk left over Q_l u P, plus the P lift (P c0, P c1), then ModDown and rescale
        as one division by P q_l."""
        if len(a.c) != 3:
            raise ValueError("relin needs a 3-poly ciphertext")
        if self.rlk is None:
            raise KeyError("missing relinearisation key")
        if a.level == 0:
            raise DepthError("depth exhausted")
        self._rec("relin_rescale", a.level)
        P = self.P
        l = a.level
        basis = self.pq_basis(l)
        nkey = P.L + 1 + P.K
        acc0 = np.zeros((l + 1 + P.K, P.n), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for j in range(-(-(l + 1) // P.alpha)):
            y = np.empty((l + 1 + P.K, P.n), dtype=np.uint64)
            lib().or_modup(P.n, l, _arr(P.q), P.K, _arr(P.p), P.alpha, j, _arr(a.c[2]), y)
            kb = np.concatenate([self.rlk[j, 0, : l + 1], self.rlk[j, 0, P.L + 1: nkey]])
            ka = np.concatenate([self.rlk[j, 1, : l + 1], self.rlk[j, 1, P.L + 1: nkey]])
            acc0 = poly_add(basis, acc0, poly_mul(basis, y, kb))
            acc1 = poly_add(basis, acc1, poly_mul(basis, y, ka))
        pm = self._p_mod(basis)
        acc0[: l + 1] = poly_add(basis[: l + 1], acc0[: l + 1], poly_scalar(basis[: l + 1], a.c[0], pm[: l + 1]))
        acc1[: l + 1] = poly_add(basis[: l + 1], acc1[: l + 1], poly_scalar(basis[: l + 1], a.c[1], pm[: l + 1]))
        return Ct([self.moddown_rescale_poly(acc0, l), self.moddown_rescale_poly(acc1, l)], l - 1,
                  a.scale / P.q[l], a.n_slots)

    def _ip_pq(self, x: np.ndarray, level: int, evk: np.ndarray):
        """The key inner product of ModUp(x) with evk left over Q_l u P (no ModDown)."""
        P = self.P
        basis = self.pq_basis(level)
        nkey = P.L + 1 + P.K
        acc0 = np.zeros((level + 1 + P.K, P.n), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for j in range(-(-(level + 1) // P.alpha)):
            y = np.empty((level + 1 + P.K, P.n), dtype=np.uint64)
            lib().or_modup(P.n, level, _arr(P.q), P.K, _arr(P.p), P.alpha, j, _arr(x), y)
            kb = np.concatenate([evk[j, 0, : level + 1], evk[j, 0, P.L + 1: nkey]])
            ka = np.concatenate([evk[j, 1, : level + 1], evk[j, 1, P.L + 1: nkey]])
            acc0 = poly_add(basis, acc0, poly_mul(basis, y, kb))
            acc1 = poly_add(basis, acc1, poly_mul(basis, y, ka))
        return acc0, acc1

    def conj_mul_relin_rescale(self, a: Ct) -> Ct:
        """d * Conj(d), relinearised and rescaled with ONE division by P q_l (reading R32): with
        sigma = sigma_{2N-1}, the product (a0 + a1 s)(sigma a0 + sigma a1 sigma s) has the terms
        t0 = a0 sigma(a0), t1 = a1 sigma(a0) (times s), t2 = a0 sigma(a1) (times sigma s) and
        t3 = a1 sigma(a1) (times s sigma s); the inner products of ModUp(t2) with the conjugation key
        and of ModUp(t3) with the conjugate-product key are summed over Q_l u P with the P lift of
        (t0, t1), then divided by P q_l (or_moddown_rescale).  Slots: |d|^2; scale s_d^2 / q_l."""
        if len(a.c) != 2:
            raise ValueError("needs a 2-poly ciphertext")
        for k in (CONJ, CONJ_PROD):
            if k not in self.gk:
                raise KeyError("missing conjugation key" if k == CONJ else "missing conjugate-product key")
        if a.level == 0:
            raise DepthError("depth exhausted")
        self._rec("conj_mul_relin_rescale", a.level)
        P = self.P
        l = a.level
        qs = self.qs(l)
        g = 2 * P.n - 1
        s0, s1 = automorphism(qs, a.c[0], g), automorphism(qs, a.c[1], g)
        t0, t1 = poly_mul(qs, a.c[0], s0), poly_mul(qs, a.c[1], s0)
        t2, t3 = poly_mul(qs, a.c[0], s1), poly_mul(qs, a.c[1], s1)
        u0, u1 = self._ip_pq(t2, l, self.gk[CONJ])
        v0, v1 = self._ip_pq(t3, l, self.gk[CONJ_PROD])
        basis = self.pq_basis(l)
        acc0, acc1 = poly_add(basis, u0, v0), poly_add(basis, u1, v1)
        pm = self._p_mod(basis)
        acc0[: l + 1] = poly_add(qs, acc0[: l + 1], poly_scalar(qs, t0, pm[: l + 1]))
        acc1[: l + 1] = poly_add(qs, acc1[: l + 1], poly_scalar(qs, t1, pm[: l + 1]))
        return Ct([self.moddown_rescale_poly(acc0, l), self.moddown_rescale_poly(acc1, l)], l - 1,
                  a.scale * a.scale / P.q[l], a.n_slots)

    def moddown_ct(self, a: Ct) -> Ct:
        """Both polynomials of a PQ ciphertext back to Q_l (divides out P)."""
        self._rec("moddown", a.level)
        return Ct([self.moddown_poly(x, a.level) for x in a.c], a.level, a.scale, a.n_slots)

    def rescale(self, a: Ct) -> Ct:
        """Divide by q_level with the pinned round-half-up rule (c-5)."""
        if len(a.c) != 2:
            raise ValueError("rescale needs a 2-poly ciphertext")
        if a.level == 0:
            raise DepthError("depth exhausted")
        self._rec("rescale", a.level)
        P = self.P
        l = a.level
        qs = _arr(P.q[: l + 1])
        out = []
        for x in a.c:
            y = np.empty((l, P.n), dtype=np.uint64)
            lib().or_rescale(P.n, l, qs, _arr(x), y)
            out.append(y)
        return Ct(out, l - 1, a.scale / P.q[l], a.n_slots)

    # --- composites
    def mul_relin(self, a: Ct, b: Ct) -> Ct:
        return self.relin(self.tensor(a, b))

    def mul_rescale(self, a: Ct, b: Ct) -> Ct:
        return self.rescale(self.relin(self.tensor(a, b)))

    def square_rescale(self, a: Ct) -> Ct:
        return self.mul_rescale(a, a)

    def rotsum(self, a: Ct, count: int, stride: int = 1) -> Ct:
        """sum_{i<count} Rot(a, i*stride) for count a power of two, by log2(count)
        rotate-and-add steps with strides stride*2^i."""
        acc = a
        step = stride
        c = 1
        while c < count:
            acc = self.add(acc, self.rotate(acc, step))
            step *= 2
            c *= 2
        return acc
