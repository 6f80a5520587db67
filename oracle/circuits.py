"""The mmFHE kernel circuits over the O-RNS evaluator -- TEST INFRASTRUCTURE ONLY.

Each function follows the paper's kernel in the paper's order and notation,
with the canonical circuit pinned in SURVEY §8(c)-7 (relinearisation
placement, rescale placement, BSGS split, overflow folds).  The CUDA library
implements the same logical op sequence independently (csrc/chains.cpp);
``op trace`` equality plus bit-exact residues is the parity gate.

Per-frame kernels take LISTS of frame ciphertexts and apply each op to every
frame before the next op ("op-major" order, one list comprehension per op).
This is only an evaluation order: each ciphertext goes through exactly the
paper's op sequence; the order fixes the trace the GPU's batched launches
reproduce.  Frames are processed in batches of ``cfg.frame_batch``.

Kernels:
  K1 Energy Integration              Eq. energy
  K2 Soft Power Attention            Eqs. soft_power_weight/soft_argmax_stats P:777-788
  K2b Doppler soft power             Eq. gesture_soft_power
  K3 Block-diagonal DFT, BSGS        Eqs. dft_kernel/dft_re P:797-815, BSGS P:164-176
  K4 Soft I/Q                        Eqs. phase_mask/phase_iq P:821-829
  K5 FIR (Toeplitz)                  Eq. fir_iq
  K6 Notch mask                      Eq. notch_mask
  K7 Taylor differential phase       Eq. taylor_arctan
  FC square-activation MLP           Eq. mlp_forward
Pipelines: vital signs P:901-902, dynamic classification P:904-907,
Table tab:depth P:914-949.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from oracle import ckks as orc
from oracle import dsp


@dataclass
class ChainCfg:
    R: int = 64
    D: int = 32
    A: int = 4
    F: int = 32
    gamma: int = 2              # K2 sharpening exponent (power of two)
    p_phi: int = 2              # K4 mask exponent (reading #1)
    taylor_order: int = 1       # K7: 1 (evaluated variant) or 3
    n_slots: int = 0            # packing period n
    bsgs_baby: int = 0          # K3 baby steps b; 0 -> ceil(sqrt(2D-1))
    fc_dims: tuple = (4096, 64, 32, 8)
    notch_width: int = 1
    fs: float = 20.0
    bands: tuple = ((0.1, 0.6), (0.8, 2.5))   # RR, HR
    frame_batch: int = 0        # frames per op-major batch (0: all frames)
    hoist: int = 0              # 1: baby-step rotations of K3 / FC share one ModUp (hoisted HRot)
    vp_plus: int = 0            # vital V2: 1 -> sharpen + weighted frequency average in the cloud
    iq_pack: int = 0            # K4: k >= 1 -> packed rotate-and-sum over 2^k vectors (reading R19)
    n_taps: tuple = ()          # k5_fir_rot: taps per band (rotation keys for the longest)
    lanes: int = 1              # gesture / K3: frames interleaved per ciphertext (reading R20)
    fc_baby: int = 0            # FC BSGS baby steps (0: ceil(sqrt(h)))
    bsgs_aligned: int = 0       # K3: 1 -> giant offsets at multiples of b, one giant step the identity (R29)
    rotsum_inner: int = 0       # double hoisting: size of the rotate-and-sum's hoisted first level (R27; 0 -> 8)
    rotsum_hoist_all: int = 0   # double hoisting: 1 -> every rotate-and-sum level hoisted (groups of rotsum_inner, R30)
    ks_merge: int = 0           # gesture / K3 / FC / vital V1, V2: 1 -> every ModDown or relinearisation followed
                                # by a rescale is ONE division by P q_l (R31)
    k1_conj_fuse: int = 0       # complex slots + ks_merge: 1 -> K1's d Conj(d) as one conjugate-product key switch
                                # (R32; needs the CONJ_PROD key)
    cplx: int = 0               # gesture / K3: 1 -> complex slots, z = v_re + j v_im in ONE ciphertext
                                # per frame (group); K3 multiplies complex diagonals, K1 is z conj(z)
                                # (reading R28)


def log2_exact(x: int, name: str) -> int:
    """log2 of a power-of-two public exponent (the number of squarings, P:777-788,
    P:821-829); anything else is rejected rather than rounded."""
    if x < 1 or x & (x - 1):
        raise ValueError(f"{name} must be a power of two, got {x}")
    return x.bit_length() - 1


def rot(v: np.ndarray, k: int) -> np.ndarray:
    """Rot(v, k)[j] = v[(j + k) mod n] (left rotation)."""
    return np.roll(v, -k)


# ------------------------------------------------------------------ SIMD-dense lanes (reading R20)
# With cfg.lanes = L > 1, one ciphertext carries L frames interleaved: slot L*i + f holds
# element i (< n) of frame f (< L).  Rot(x, L k)[L i + f] = x[L (i + k) + f] (mod n L), so
# every per-frame rotation by k becomes a slot rotation by L k, every public plaintext
# vector p (period n) becomes p repeated L times per entry, and lanes never mix.  The
# frames' features are summed across lanes (rotate-and-sum, strides 1 .. L/2) before the
# classifier's first nonlinearity; the logits then sit in slots L c.  SURVEY §8(f)-3.

def lanes_of(cfg) -> int:
    L = int(getattr(cfg, "lanes", 1) or 1)
    log2_exact(L, "lanes")
    return L


def lane_vec(v: np.ndarray, L: int) -> np.ndarray:
    """A per-frame public vector in the lane-interleaved layout (entry i in slots L i .. L i + L-1)."""
    v = np.asarray(v)
    return np.repeat(v, L) if L > 1 else v


def interleave(frames, L: int, n: int) -> np.ndarray:
    """Client packing: up to L frame vectors of length n into one slot vector (unused lanes 0);
    complex frames give a complex slot vector (reading R28)."""
    out = np.zeros(n * L, dtype=np.complex128 if any(np.iscomplexobj(v) for v in frames) else np.float64)
    for f, v in enumerate(frames):
        out[f::L] = v
    return out


def n_packed(F: int, L: int) -> int:
    """Ciphertext pairs holding F frames at L frames per ciphertext."""
    return -(-F // L)


def logit_slots(n_classes: int, L: int) -> list:
    return [c * L for c in range(n_classes)]


def ceil_sqrt(x: int) -> int:
    return int(math.ceil(math.sqrt(x)))


def chunks(n: int, size: int):
    size = size or n
    return [(s, min(n, s + size)) for s in range(0, n, size)]


class PlainBook:
    """Public plaintext operands encoded by the oracle at the level
    they are used, Delta_pt = q_level unless a scale is given.  Parity mode
    imports exactly these residues into the GPU context by (name, level)."""

    def __init__(self, P):
        self.P = P
        self.entries: dict = {}
        self.encode_s = 0.0  # seconds spent encoding (setup work; bench.py excludes it)

    def vec(self, name: str, values: np.ndarray, level: int, scale: float | None = None):
        key = (name, level)
        if key not in self.entries:
            t0 = time.perf_counter()
            sc = float(self.P.q[level]) if scale is None else float(scale)
            self.entries[key] = (orc.encode(self.P, values, sc, level), sc, np.asarray(values))
            self.encode_s += time.perf_counter() - t0
        res, sc, _ = self.entries[key]
        return res, sc

    def vec_pq(self, name: str, values: np.ndarray, level: int):
        """The same encoding over Q_level u P (double-hoisted BSGS diagonals), stored under
        (name + ".pq", level); Delta_pt = q_level."""
        key = (name + ".pq", level)
        if key not in self.entries:
            t0 = time.perf_counter()
            sc = float(self.P.q[level])
            self.entries[key] = (orc.encode_pq(self.P, values, sc, level), sc, np.asarray(values))
            self.encode_s += time.perf_counter() - t0
        res, sc, _ = self.entries[key]
        return res, sc


# ------------------------------------------------------------------ evaluator ext

class CircuitEvaluator(orc.Evaluator):
    """Logical ops used by the circuits, each recorded once in the trace.  merge_rescale (set by the
    gesture / K3 / FC entry points from cfg.ks_merge, reading R31): relinearisation + rescale and
    ModDown + rescale run as one division by P q_l."""

    merge_rescale = False

    def tensor_sum(self, pairs) -> orc.Ct:
        """sum_i tensor(a_i, b_i) -- the lazy-relinearisation input (c-6)."""
        a0 = pairs[0][0]
        self._rec("tensor_sum", a0.level, str(len(pairs)))
        qs = self.qs(a0.level)
        acc = None
        for a, b in pairs:
            if a.level != b.level or a.level != a0.level:
                raise ValueError("level mismatch")
            d0 = orc.poly_mul(qs, a.c[0], b.c[0])
            d1 = orc.poly_add(qs, orc.poly_mul(qs, a.c[0], b.c[1]), orc.poly_mul(qs, a.c[1], b.c[0]))
            d2 = orc.poly_mul(qs, a.c[1], b.c[1])
            t = [d0, d1, d2]
            acc = t if acc is None else [orc.poly_add(qs, x, y) for x, y in zip(acc, t)]
        sc = pairs[0][0].scale * pairs[0][1].scale
        for a, b in pairs:
            if a.scale * b.scale != sc:
                raise orc.ScaleError("tensor_sum scale mismatch")
        return orc.Ct(acc, a0.level, sc, a0.n_slots)

    def pmult_sum(self, terms) -> orc.Ct:
        """sum_i pt_i (.) ct_i, all at one level and equal products of scales."""
        ct0 = terms[0][1]
        self._rec("pmult_sum", ct0.level, str(len(terms)))
        qs = self.qs(ct0.level)
        acc = None
        sc = None
        for (pt, pts), ct in terms:
            if ct.level != ct0.level:
                raise ValueError("level mismatch")
            t = [orc.poly_mul(qs, x, pt[: ct.level + 1]) for x in ct.c]
            acc = t if acc is None else [orc.poly_add(qs, x, y) for x, y in zip(acc, t)]
            s = ct.scale * pts
            if sc is None:
                sc = s
            elif s != sc:
                raise orc.ScaleError("pmult_sum scale mismatch")
        return orc.Ct(acc, ct0.level, sc, ct0.n_slots)

    def pmult_sum_pq(self, terms) -> orc.Ct:
        """sum_i pt_i (.) ct_i over Q_l u P (PQ ciphertexts and PQ-encoded plaintexts)."""
        ct0 = terms[0][1]
        self._rec("pmult_sum_pq", ct0.level, str(len(terms)))
        basis = self.pq_basis(ct0.level)
        acc = None
        sc = None
        for (pt, pts), ct in terms:
            t = [orc.poly_mul(basis, x, pt) for x in ct.c]
            acc = t if acc is None else [orc.poly_add(basis, x, y) for x, y in zip(acc, t)]
            s = ct.scale * pts
            if sc is None:
                sc = s
            elif s != sc:
                raise orc.ScaleError("pmult_sum_pq scale mismatch")
        return orc.Ct(acc, ct0.level, sc, ct0.n_slots)

    def lincomb_scalar(self, cts, coefs) -> orc.Ct:
        """sum_k round-half-away(c_k q_l) ct_k (exact scalar encoding, c-5)."""
        ct0 = cts[0]
        self._rec("lincomb", ct0.level, str(len(cts)))
        qs = self.qs(ct0.level)
        ql = self.P.q[ct0.level]
        acc = None
        for ct, c in zip(cts, coefs):
            if ct.level != ct0.level or ct.scale != ct0.scale:
                raise orc.ScaleError("lincomb operands must share level and scale")
            v = orc.encode_scalar(float(c), ql)
            res = np.array([v % q for q in qs], dtype=np.uint64)
            t = [orc.poly_scalar(qs, x, res) for x in ct.c]
            acc = t if acc is None else [orc.poly_add(qs, x, y) for x, y in zip(acc, t)]
        return orc.Ct(acc, ct0.level, ct0.scale * ql, ct0.n_slots)

    def add_plain(self, ct: orc.Ct, pt) -> orc.Ct:
        res, sc = pt
        if sc != ct.scale:
            raise orc.ScaleError("add_plain scale mismatch")
        self._rec("add_plain", ct.level)
        qs = self.qs(ct.level)
        return orc.Ct([orc.poly_add(qs, ct.c[0], res[: ct.level + 1]), ct.c[1]], ct.level, ct.scale, ct.n_slots)

    # ---- op-major helpers over frame lists
    def relin_rescale_all(self, cts):
        if self.merge_rescale:
            return [self.relin_rescale_merged(x) for x in cts]
        return [self.rescale(x) for x in [self.relin(x) for x in cts]]

    def down_rescale(self, x):
        """A PQ ciphertext's ModDown followed by the rescale (one division with merge_rescale, R31)."""
        return self.moddown_rescale_ct(x) if self.merge_rescale else self.rescale(self.moddown_ct(x))

    def square_rescale_all(self, cts):
        return self.relin_rescale_all([self.tensor_sum([(x, x)]) for x in cts])

    def rotsum_all(self, cts, count: int, stride: int):
        """sum_{i<count} Rot(x, i*stride) for every x: log2(count) rotate-and-add
        steps with strides stride*2^i."""
        acc = list(cts)
        step, c = stride, 1
        while c < count:
            r = [self.rotate(x, step) for x in acc]
            acc = [self.add(x, y) for x, y in zip(acc, r)]
            step *= 2
            c *= 2
        return acc


    def rotsum_dh_all(self, cts, count: int, stride: int, inner: int = 8, all_levels: bool = False):
        """Rotate-and-sum with a double-hoisted first level (reading R27):
        with a = min(inner, count), t = ModDown(P x + sum_{0<j<a} Rot_PQ(x, j stride)) -- one
        ModUp of x, a - 1 hoisted rotations left over Q_l u P (hoisted_step_pq), their PQ sum
        and one ModDown -- then the remaining log2(count / a) rotate-and-add steps with
        strides a stride 2^i.  The same slot sums as rotsum_all (decryption), other residues.
        Op-major: the lifts, every rotation (step-major), then the PQ additions."""
        a = min(inner, count)
        if a <= 1:
            return self.rotsum_all(cts, count, stride)
        ys = [self.hoist_modup(x) for x in cts]
        acc = [self.lift_pq(x) for x in cts]
        rots = [[self.hoisted_step_pq(x, y, stride * j) for x, y in zip(cts, ys)] for j in range(1, a)]
        for r in rots:
            acc = [self.add_pq(p, q) for p, q in zip(acc, r)]
        t = [self.moddown_ct(p) for p in acc]
        if all_levels and count // a > 1:
            # reading R30: the remaining sum is again a double-hoisted level (groups of `inner`)
            return self.rotsum_dh_all(t, count // a, stride * a, inner, True)
        return self.rotsum_all(t, count // a, stride * a)


# ------------------------------------------------------------------ K1 / K2

def k1_energy(ev: CircuitEvaluator, re_list, im_list) -> orc.Ct:
    """K1: E = rescale(relin(sum_t tensor(re_t,re_t) + tensor(im_t,im_t)))."""
    pairs = []
    for re, im in zip(re_list, im_list):
        pairs += [(re, re), (im, im)]
    return ev.relin_rescale_all([ev.tensor_sum(pairs)])[0]


def k1_energy_sessions(ev: CircuitEvaluator, sessions):
    """K1 for several independent sessions [(re_list, im_list), ...], op-major."""
    ts = []
    for re_list, im_list in sessions:
        pairs = []
        for re, im in zip(re_list, im_list):
            pairs += [(re, re), (im, im)]
        ts.append(ev.tensor_sum(pairs))
    return ev.relin_rescale_all(ts)


def k2_soft_attention(ev: CircuitEvaluator, book: PlainBook, E: orc.Ct, cfg: ChainCfg):
    """K2a: w = E^gamma by log2(gamma) squarings; N = rotsum_R(w (.) ramp'),
    D = rotsum_R(w (.) one'), ramp'_r = r/(F^2 R), one'_r = 1/(F^2 R)."""
    w = E
    for _ in range(log2_exact(cfg.gamma, "gamma")):
        w = ev.square_rescale_all([w])[0]
    n = E.n_slots
    R, F = cfg.R, cfg.F
    ramp = np.zeros(n)
    one = np.zeros(n)
    ramp[:R] = np.arange(R) / (F * F * R)
    one[:R] = 1.0 / (F * F * R)
    Nn = ev.rescale(ev.pmult_sum([(book.vec("k2.ramp", ramp, w.level), w)]))
    Dd = ev.rescale(ev.pmult_sum([(book.vec("k2.one", one, w.level), w)]))
    return ev.rotsum_all([Nn], R, 1)[0], ev.rotsum_all([Dd], R, 1)[0]


def vitals_v1(ev, book, re_list, im_list, cfg):
    """Chain V1 = K1 -> K2; the client decrypts N and D, r_hat = N/D."""
    set_merge(ev, cfg)
    return k2_soft_attention(ev, book, k1_energy(ev, re_list, im_list), cfg)


# ------------------------------------------------------------------ K3 (BSGS)

def block_diag_diagonal(M: np.ndarray, n: int, o: int) -> np.ndarray:
    """diag_o of I_{n/D} (x) M: diag_o[j] = Mt[j, (j+o) mod n] (Halevi-Shoup)."""
    D = M.shape[0]
    out = np.zeros(n, dtype=M.dtype)
    for j in range(n):
        c = (j + o) % n
        if j // D == c // D:
            out[j] = M[j % D, c % D]
    return out


def k3_schedule(cfg: ChainCfg):
    """BSGS split over the offsets o in [-(D-1), D-1]: o = o_min + g'b + s, or with
    cfg.bsgs_aligned (reading R29) o = G + s with giant offsets G = b k, k = floor(-(D-1)/b) ..
    floor((D-1)/b): the giant G = 0 needs no rotation (one giant key switch fewer per input)."""
    D = cfg.D
    d = 2 * D - 1
    b = cfg.bsgs_baby or ceil_sqrt(d)
    giants = []
    if getattr(cfg, "bsgs_aligned", 0):
        for gp, k in enumerate(range(-((D - 1 + b - 1) // b), (D - 1) // b + 1)):
            G = b * k
            giants.append((gp, G, [s for s in range(b) if -(D - 1) <= G + s <= D - 1]))
        return b, giants
    g = -(-d // b)
    o_min = -(D - 1)
    for gp in range(g):
        G = o_min + gp * b
        babies = [s for s in range(b) if G + s <= D - 1]
        giants.append((gp, G, babies))
    return b, giants


def k3_prefix(cfg) -> str:
    """Plaintext-name prefix of K3's diagonals (the aligned schedule's differ, R29)."""
    return "k3a" if getattr(cfg, "bsgs_aligned", 0) else "k3"


def baby_steps(ev, cts, steps, hoist):
    """[[Rot(x, s) for x in cts] for s in steps]: plain HRots, or hoisted HRots that
    share one ModUp per ciphertext (SURVEY §8(c)-5 'Hoisted HRot is a different op'),
    or (hoist = 2, double hoisting) hoisted rotations left over Q_l u P."""
    if not hoist:
        return [[ev.rotate(x, s) for x in cts] for s in steps]
    ys = [ev.hoist_modup(x) for x in cts]
    if hoist == 2:
        return [[ev.hoisted_step_pq(x, y, s) for x, y in zip(cts, ys)] for s in steps]
    return [[ev.hoisted_step(x, y, s) for x, y in zip(cts, ys)] for s in steps]


def rotsum_inner(cfg) -> int:
    """Size a of the double-hoisted first rotate-and-sum level (R27): cfg.rotsum_inner, a power of
    two (0 -> 8)."""
    a = int(getattr(cfg, "rotsum_inner", 0) or 8)
    log2_exact(a, "rotsum_inner")
    return a


def rotsum_dh(ev, cts, count: int, stride: int, cfg, inner: int | None = None):
    """The rotate-and-sum of the double-hoisted circuits: rotsum_dh_all with the chain's level size
    (R27) and, with cfg.rotsum_hoist_all, every level hoisted (R30)."""
    return ev.rotsum_dh_all(cts, count, stride, rotsum_inner(cfg) if inner is None else inner,
                            bool(getattr(cfg, "rotsum_hoist_all", 0)))


def rotsum_levels(count: int, inner: int, all_levels: bool):
    """Group sizes of the double-hoisted levels of a rotate-and-sum over `count` terms (R27 / R30);
    the plain rotate-and-add steps that follow the hoisted levels are log2 of what is left."""
    out, c = [], count
    while c > 1:
        a = min(inner, c)
        out.append(a)
        c //= a
        if not all_levels:
            break
    return out


def k1_fused(cfg) -> bool:
    """Reading R32: K1's d Conj(d) as one conjugate-product key switch (complex slots with ks_merge)."""
    if not getattr(cfg, "k1_conj_fuse", 0):
        return False
    if not (cplx_of(cfg) and getattr(cfg, "ks_merge", 0)):
        raise ValueError("k1_conj_fuse needs complex slots (cplx) and ks_merge")
    return True


def set_merge(ev, cfg):
    """Reading R31 for the gesture / K3 / FC and vital (V1 / V2) chains: the evaluator merges every relinearisation or
    ModDown that a rescale follows into one division by P q_l (cfg.ks_merge)."""
    ev.merge_rescale = bool(getattr(cfg, "ks_merge", 0))


def dh(cfg) -> bool:
    """Double-hoisted BSGS (cfg.hoist = 2): baby steps stay over
    Q_l u P (no ModDown), the inner sums multiply PQ-encoded diagonals, every giant step
    ModDowns only its inner sum's second polynomial before its key switch and keeps the
    result over Q_l u P, and one ModDown per output ends the giant sum."""
    return getattr(cfg, "hoist", 0) == 2


def cplx_of(cfg) -> bool:
    """Complex-slot packing (reading R28): one ciphertext z = v_re + j v_im per frame (group)."""
    return bool(getattr(cfg, "cplx", 0))


def k3_babies(ev: CircuitEvaluator, v, cfg: ChainCfg):
    """[x, Rot(x, s L)] for s < b and every x of the frame list v (the identity step lifted
    to Q_l u P under double hoisting)."""
    L = lanes_of(cfg)
    n = v[0].n_slots // L
    if n % cfg.D or n < 2 * cfg.D:
        # the 2D-1 offsets of the block-diagonal matrix alias when a period holds one block
        raise ValueError("K3 needs the packing period to be a multiple of D and at least 2D")
    b, _ = k3_schedule(cfg)
    if dh(cfg):
        return [[ev.lift_pq(x) for x in v]] + baby_steps(ev, v, [s * L for s in range(1, b)], 2)
    return [list(v)] + baby_steps(ev, v, [s * L for s in range(1, b)], cfg.hoist)


def k3_baby_steps(ev: CircuitEvaluator, v_re, v_im, cfg: ChainCfg):
    """K3 BSGS baby steps: [x, Rot(x, s)] for s < b, for v_re and v_im."""
    xr = k3_babies(ev, v_re, cfg)
    xi = k3_babies(ev, v_im, cfg)
    return xr, xi


def k3_inner_sums(ev: CircuitEvaluator, book: PlainBook, xr, xi, cfg: ChainCfg):
    """Every giant step's inner sums (one pass over the baby steps): for giant g',
    d_re part sum_s C~'_{g',s} Rot(v_re, s) - S~'_{g',s} Rot(v_im, s) and the d_im part
    sum_s S~'_{g',s} Rot(v_re, s) + C~'_{g',s} Rot(v_im, s), with the diagonals of
    Eqs. dft_re / dft_im pre-rotated by -G (Halevi-Shoup)."""
    L = lanes_of(cfg)
    n = xr[0][0].n_slots // L
    lvl = xr[0][0].level
    W = dsp.dft_matrix(cfg.D)
    C, S = W.real, W.imag
    _, giants = k3_schedule(cfg)
    nf = len(xr[0])

    def terms(spec, f):
        return [(pt, (xr if which == "r" else xi)[s][f]) for pt, s, which in spec]

    inner = []
    for gp, G, babies in giants:
        t_re, t_im = [], []
        for s in babies:
            o = G + s
            dc = lane_vec(rot(block_diag_diagonal(C, n, o), -G), L)
            ds = lane_vec(rot(block_diag_diagonal(S, n, o), -G), L)
            vec = book.vec_pq if dh(cfg) else book.vec
            pc = vec(f"{k3_prefix(cfg)}.c.{gp}.{s}", dc, lvl)
            ps = vec(f"{k3_prefix(cfg)}.s.{gp}.{s}", ds, lvl)
            pns = vec(f"{k3_prefix(cfg)}.ns.{gp}.{s}", -ds, lvl)
            t_re += [(pc, s, "r"), (pns, s, "i")]
            t_im += [(ps, s, "r"), (pc, s, "i")]
        psum = ev.pmult_sum_pq if dh(cfg) else ev.pmult_sum
        inner.append(([psum(terms(t_re, f)) for f in range(nf)],
                      [psum(terms(t_im, f)) for f in range(nf)]))
    return inner


def k3_giant_steps(ev: CircuitEvaluator, inner, cfg: ChainCfg):
    """Giant rotations Rot(inner_g', G) summed over g', one rescale after the sum (c-6)."""
    L = lanes_of(cfg)
    _, giants = k3_schedule(cfg)
    out_re = out_im = None
    rot, add = (ev.rotate_pq, ev.add_pq) if dh(cfg) else (ev.rotate, ev.add)
    for (gp, G, babies), (pr, pi) in zip(giants, inner):
        ir = [rot(x, G * L) for x in pr]
        ii = [rot(x, G * L) for x in pi]
        out_re = ir if out_re is None else [add(a, x) for a, x in zip(out_re, ir)]
        out_im = ii if out_im is None else [add(a, x) for a, x in zip(out_im, ii)]
    if dh(cfg) and ev.merge_rescale:
        return [ev.down_rescale(x) for x in out_re], [ev.down_rescale(x) for x in out_im]
    if dh(cfg):
        out_re = [ev.moddown_ct(x) for x in out_re]
        out_im = [ev.moddown_ct(x) for x in out_im]
    return [ev.rescale(x) for x in out_re], [ev.rescale(x) for x in out_im]


def k3_doppler_dft_frames(ev: CircuitEvaluator, book: PlainBook, v_re, v_im, cfg: ChainCfg):
    """K3 (Eqs. dft_re/dft_im P:805-815) on a list of frames: d_re = C~ v_re - S~ v_im,
    d_im = S~ v_re + C~ v_im via BSGS with pre-rotated diagonals: baby steps, all giant
    steps' inner sums, then the giant rotations; one rescale after the giant sum (c-6)."""
    set_merge(ev, cfg)
    xr, xi = k3_baby_steps(ev, v_re, v_im, cfg)
    return k3_giant_steps(ev, k3_inner_sums(ev, book, xr, xi, cfg), cfg)


def k3_inner_sums_c(ev: CircuitEvaluator, book: PlainBook, xs, cfg: ChainCfg):
    """Complex slots (reading R28): every giant step's inner sum sum_s W~'_{g',s} Rot(z, s)
    with the complex diagonals of W~ = I_{AR} (x) W (Eq. dft_kernel; Eq. dft_re's
    d_re + j d_im = (C~ + j S~)(v_re + j v_im)) pre-rotated by -G -- one product
    per (giant, baby), the complex multiplication done by the slot-wise plaintext product."""
    L = lanes_of(cfg)
    n = xs[0][0].n_slots // L
    lvl = xs[0][0].level
    W = dsp.dft_matrix(cfg.D)
    _, giants = k3_schedule(cfg)
    nf = len(xs[0])
    vec = book.vec_pq if dh(cfg) else book.vec
    psum = ev.pmult_sum_pq if dh(cfg) else ev.pmult_sum
    inner = []
    for gp, G, babies in giants:
        pts = [(vec(f"{k3_prefix(cfg)}.w.{gp}.{s}", lane_vec(rot(block_diag_diagonal(W, n, G + s), -G), L), lvl), s)
               for s in babies]
        inner.append([psum([(pt, xs[s][f]) for pt, s in pts]) for f in range(nf)])
    return inner


def k3_giant_steps_c(ev: CircuitEvaluator, inner, cfg: ChainCfg):
    """Giant rotations of the complex inner sums, summed, one ModDown (double hoisting) and
    one rescale after the sum (c-6)."""
    L = lanes_of(cfg)
    _, giants = k3_schedule(cfg)
    out = None
    rot_, add = (ev.rotate_pq, ev.add_pq) if dh(cfg) else (ev.rotate, ev.add)
    for (gp, G, babies), pr in zip(giants, inner):
        r = [rot_(x, G * L) for x in pr]
        out = r if out is None else [add(a, x) for a, x in zip(out, r)]
    if dh(cfg) and ev.merge_rescale:
        return [ev.down_rescale(x) for x in out]
    if dh(cfg):
        out = [ev.moddown_ct(x) for x in out]
    return [ev.rescale(x) for x in out]


def k3_doppler_dft_frames_c(ev: CircuitEvaluator, book: PlainBook, z, cfg: ChainCfg):
    """K3 on complex-slot frames (reading R28): d = W~ z by BSGS, d in complex slots."""
    set_merge(ev, cfg)
    return k3_giant_steps_c(ev, k3_inner_sums_c(ev, book, k3_babies(ev, z, cfg), cfg), cfg)


def k3_doppler_dft(ev, book, v_re, v_im, cfg):
    """K3 on one frame."""
    dre, dim = k3_doppler_dft_frames(ev, book, [v_re], [v_im], cfg)
    return dre[0], dim[0]


# ------------------------------------------------------------------ gesture frame

def k1_power(ev, d_re, d_im):
    """K1 on the K3 output: P = rescale(relin(tensor(d_re,d_re) + tensor(d_im,d_im)))."""
    return ev.relin_rescale_all([ev.tensor_sum([(a, a), (b, b)]) for a, b in zip(d_re, d_im)])


def k1_power_c(ev, d, fuse=False):
    """K1 on complex-slot K3 outputs (reading R28): P = rescale(relin(tensor(d, Conj(d)))),
    d conj(d) = d_re^2 + d_im^2 in every slot (Eq. energy's |.|^2); with fuse (R32) the
    conjugation and the relinearisation share one division (Evaluator.conj_mul_relin_rescale)."""
    if fuse:
        return [ev.conj_mul_relin_rescale(x) for x in d]
    cj = [ev.conjugate(x) for x in d]
    return ev.relin_rescale_all([ev.tensor_sum([(a, b)]) for a, b in zip(d, cj)])


def k6_notch(ev, book, P_cts, cfg):
    """K6: P (.) m~ with m~[d] = m[d]/s, s = R A (sum w)^2 (P:887 fold)."""
    L = lanes_of(cfg)
    n = P_cts[0].n_slots // L
    s = dsp.spectral_scale(cfg.R, cfg.A, cfg.D)
    mask = lane_vec(np.tile(dsp.notch_mask(cfg.D, cfg.notch_width) / s, n // cfg.D), L)
    pt = book.vec("k6.mask", mask, P_cts[0].level)
    return [ev.rescale(x) for x in [ev.pmult_sum([(pt, p)]) for p in P_cts]]


def k2_doppler_soft_power(ev, Pm, cfg):
    """K2b (Eq. gesture_soft_power): S = rotsum over the n/D blocks
    (stride D; every block then holds sum_{a,r}, reading #8); S^gamma by squarings;
    f = Pm (.) S^gamma (P:906 'feature weighting')."""
    L = lanes_of(cfg)
    count, stride = Pm[0].n_slots // L // cfg.D, cfg.D * L
    S = rotsum_dh(ev, Pm, count, stride, cfg) if dh(cfg) else ev.rotsum_all(Pm, count, stride)
    for _ in range(log2_exact(cfg.gamma, "gamma")):
        S = ev.square_rescale_all(S)
    Pd = [ev.drop_to(p, s.level) for p, s in zip(Pm, S)]
    return ev.relin_rescale_all([ev.tensor_sum([(p, s)]) for p, s in zip(Pd, S)])


def gesture_frames(ev, book, v_re, v_im, cfg):
    """Per frame: K3 -> K1 -> K6 -> K2b -> weighting, on a list of frames.
    With complex slots (cfg.cplx) v_re holds the frames' z ciphertexts and v_im is None."""
    set_merge(ev, cfg)
    if cplx_of(cfg):
        if v_im is not None:
            raise ValueError("complex slots: one ciphertext per frame (v_im must be None)")
        P_cts = k1_power_c(ev, k3_doppler_dft_frames_c(ev, book, v_re, cfg), k1_fused(cfg))
    else:
        d_re, d_im = k3_doppler_dft_frames(ev, book, v_re, v_im, cfg)
        P_cts = k1_power(ev, d_re, d_im)
    Pm = k6_notch(ev, book, P_cts, cfg)
    return k2_doppler_soft_power(ev, Pm, cfg)


def gesture_frame(ev, book, v_re, v_im, cfg):
    return gesture_frames(ev, book, [v_re], None if v_im is None else [v_im], cfg)[0]


def frame_accumulate(ev, feats):
    """FA: homomorphic sum over frames (depth 0)."""
    acc = feats[0]
    for f in feats[1:]:
        acc = ev.add(acc, f)
    return acc


def gesture_features(ev, book, v_re, v_im, cfg):
    """All F frames in batches of cfg.frame_batch: per batch the frame kernels, the
    batch's features summed, batches then added in order."""
    acc = None
    for s, e in chunks(len(v_re), cfg.frame_batch):
        part = frame_accumulate(ev, gesture_frames(ev, book, v_re[s:e], None if v_im is None else v_im[s:e], cfg))
        acc = part if acc is None else ev.add(acc, part)
    return acc


# ------------------------------------------------------------------ FC

def fc_diagonal(W: np.ndarray, n_in: int, i: int) -> np.ndarray:
    """Hybrid diagonal: diag_i[j] = W[j mod h, (j+i) mod n_in], j < n_in."""
    h = W.shape[0]
    j = np.arange(n_in)
    return W[j % h, (j + i) % n_in]


def fc_schedule(h: int, fc_baby: int = 0):
    """BSGS split of an FC layer's h diagonals: b = min(fc_baby, h), or ceil(sqrt(h))."""
    b = min(fc_baby, h) if fc_baby else ceil_sqrt(h)
    g = -(-h // b)
    return b, [(gp, gp * b, [s for s in range(b) if gp * b + s < h]) for gp in range(g)]


def fc_layer(ev, book, x, W: np.ndarray, bias: np.ndarray, n_in: int, layer: int, square: bool, hoist: int = 0,
             L: int = 1, fc_baby: int = 0, rs_inner: int = 8, rs_all: bool = False):
    """One layer of Eq. mlp_forward: z = sum_i diag_i (.) Rot(x, i) by BSGS,
    y = rotsum_{n_in/h}(z, stride h) (h-periodic W x), + b, then (.)^2 unless last.
    L lanes: rotations by L i, lane-interleaved diagonals and bias (reading R20)."""
    h = W.shape[0]
    lvl = x.level
    b, giants = fc_schedule(h, fc_baby)
    pq = hoist == 2  # double-hoisted BSGS (see dh())
    babies = ([ev.lift_pq(x)] if pq else [x]) + [r[0] for r in baby_steps(ev, [x], [s * L for s in range(1, min(b, h))],
                                                                           hoist)]
    acc = None
    inners = []  # all giant steps' inner sums first, then the giant rotations
    vec = book.vec_pq if pq else book.vec
    for gp, G, ss in giants:
        terms = []
        for s in ss:
            dg = lane_vec(rot(fc_diagonal(W, n_in, G + s), -G), L)
            terms.append((vec(f"fc{layer}.d.{gp}.{s}", dg, lvl), babies[s]))
        inners.append(ev.pmult_sum_pq(terms) if pq else ev.pmult_sum(terms))
    for (gp, G, ss), inner in zip(giants, inners):
        if G:
            inner = ev.rotate_pq(inner, G * L) if pq else ev.rotate(inner, G * L)
        acc = inner if acc is None else (ev.add_pq(acc, inner) if pq else ev.add(acc, inner))
    z = ev.down_rescale(acc) if pq else ev.rescale(acc)
    y = (ev.rotsum_dh_all([z], n_in // h, h * L, rs_inner, rs_all) if pq else ev.rotsum_all([z], n_in // h, h * L))[0]
    bv = lane_vec(np.asarray(bias, dtype=np.float64), L)
    y = ev.add_plain(y, book.vec(f"fc{layer}.bias", bv, y.level, scale=y.scale))
    if square:
        y = ev.square_rescale_all([y])[0]
    return y


def pad_fc(Ws, bs, dims):
    """Pad the last layer's rows to dims[-1] (5 logits -> 8)."""
    Ws = [np.asarray(W, dtype=np.float64) for W in Ws]
    bs = [np.asarray(b, dtype=np.float64) for b in bs]
    h = dims[-1]
    if Ws[-1].shape[0] < h:
        pad = h - Ws[-1].shape[0]
        Ws[-1] = np.vstack([Ws[-1], np.zeros((pad, Ws[-1].shape[1]))])
        bs[-1] = np.concatenate([bs[-1], np.zeros(pad)])
    return Ws, bs


def gesture_fc(ev, book, feat, Ws, bs, cfg):
    """FC1 -> x^2 -> FC2 -> x^2 -> FC3.  With L lanes the frame features are
    first summed across lanes (rotate-and-sum, strides 1 .. L/2; lane 0 then holds the
    session's feature vector, reading R20) -- here rather than per partial sum, so that
    frame sharding stays an exact modular sum."""
    dims = cfg.fc_dims
    Ws, bs = pad_fc(Ws, bs, dims)
    L = lanes_of(cfg)
    set_merge(ev, cfg)
    inner = rotsum_inner(cfg)
    if L > 1:
        x = (rotsum_dh(ev, [feat], L, 1, cfg) if dh(cfg) else ev.rotsum_all([feat], L, 1))[0]
    else:
        x = feat
    for layer in range(len(Ws)):
        x = fc_layer(ev, book, x, Ws[layer], bs[layer], dims[layer], layer + 1, layer < len(Ws) - 1, cfg.hoist, L,
                     getattr(cfg, "fc_baby", 0), inner, bool(getattr(cfg, "rotsum_hoist_all", 0)))
    return x


# ------------------------------------------------------------------ vital V2

def k4_soft_iq(ev, re, im, cfg):
    """K4 on lists of frames, P_phi = 2^k: p = |z|^2, m = p^P_phi,
    i = m re, q = m im, I = rotsum_R(i), Q = rotsum_R(q) (slot 0 valid)."""
    m = ev.relin_rescale_all([ev.tensor_sum([(r, r), (i, i)]) for r, i in zip(re, im)])
    for _ in range(log2_exact(cfg.p_phi, "p_phi")):
        m = ev.square_rescale_all(m)
    red = [ev.drop_to(r, x.level) for r, x in zip(re, m)]
    i_ = ev.relin_rescale_all([ev.tensor_sum([(x, r)]) for x, r in zip(m, red)])
    imd = [ev.drop_to(i, x.level) for i, x in zip(im, m)]
    q_ = ev.relin_rescale_all([ev.tensor_sum([(x, i)]) for x, i in zip(m, imd)])
    if cfg.iq_pack:
        return k4_packed_rotsum(ev, i_, q_, cfg.R, cfg.iq_pack, cfg.hoist)
    return ev.rotsum_all(i_, cfg.R, 1), ev.rotsum_all(q_, cfg.R, 1)


def unpack_shifts(k):
    """Block order (in units of R) of the unpacked I list: [0] then, for j = k-1..1,
    seq ++ [s + 2^j for s in seq] (the order x <- x ++ Rot(x, 2^j R) produces)."""
    seq = [0]
    for j in reversed(range(1, k)):
        seq = seq + [s + (1 << j) for s in seq]
    return seq


def k4_packed_rotsum(ev, i_, q_, R, k, hoist=0):
    """Reading R19: I = rotsum_R(i), Q = rotsum_R(q) for F frames with one rotate-and-sum per
    2^(k-1) frames.  i and q occupy slots 0..R-1 (zeros beyond, reading #23).  Pack:
    x = i + Rot(q, -R) (q to slots R..2R-1), then k-1 times pair the first and second half
    of the frame list, x = x_lo + Rot(x_hi, -2^j R): 2^k vectors in slots 0..2^k R - 1.  One
    rotsum_R leaves each vector's sum in the first slot of its block.  Unpack in reverse:
    x <- x ++ Rot(x, 2^j R) (j = k-1..1), I = x, Q = Rot(x, R).  Per frame
    2 (2 - 2^(1-k)) + log2(R) / 2^(k-1) rotations instead of 2 log2 R."""
    if len(i_) % (1 << (k - 1)):
        raise ValueError("iq_pack = k needs a multiple of 2^(k-1) frames per frame batch")
    # blocks sit at multiples of R and rotsum_R adds 2^ceil(log2 R) slots: R must be 2^m,
    # or a block's sum would pick up the next block's values
    log2_exact(R, "R (iq_pack)")
    x = [ev.add(a, b) for a, b in zip(i_, [ev.rotate(v, -R) for v in q_])]
    for j in range(1, k):
        h = len(x) // 2
        lo, hi = x[:h], x[h:]
        x = [ev.add(a, b) for a, b in zip(lo, [ev.rotate(v, -(R << j)) for v in hi])]
    x = ev.rotsum_all(x, R, 1)
    if hoist:
        # every unpacking rotation acts on the packed x: one hoisted group Rot(x, mR),
        # m = 1..2^k - 1, sharing one ModUp (SURVEY §8(c)-5 hoisted HRot)
        blocks = [list(x)] + baby_steps(ev, x, [m * R for m in range(1, 1 << k)], 1)
        seq = unpack_shifts(k)
        return ([v for s in seq for v in blocks[s]], [v for s in seq for v in blocks[s + 1]])
    for j in reversed(range(1, k)):
        x = x + [ev.rotate(v, R << j) for v in x]
    return x, [ev.rotate(v, R) for v in x]


def k5_fir(ev, xs, taps):
    """K5: x_f[t] = rescale(sum_{k <= t} h[k] x[t-k]) (causal Toeplitz)."""
    lin = []
    for t in range(len(xs)):
        ks = [k for k in range(len(taps)) if t - k >= 0]
        lin.append(ev.lincomb_scalar([xs[t - k] for k in ks], [taps[k] for k in ks]))
    return [ev.rescale(x) for x in lin]


def fir_rot_schedule(W: int):
    """BSGS split of the W taps of the rotation-based FIR: k = g' b + s."""
    b = ceil_sqrt(W)
    g = -(-W // b)
    return b, [(gp, [s for s in range(b) if gp * b + s < W]) for gp in range(g)]


def k5_fir_rot(ev, x, taps, hoist=1):
    """K5 "Alternate Implementation": y[n] = sum_k h[k] x[n - k] as weighted
    accumulation over slot rotations, for a sequence packed in the slots of ONE ciphertext
    (x[t] in slot t, zeros beyond the sequence, reading #23: the rotations then bring zeros in,
    i.e. causal with zero initial state).  BSGS over the taps: baby steps Rot(x, -s) (hoisted),
    per giant g' the scalar combination sum_s h[g'b + s] Rot(x, -s) (exact encoding at q_l,
    c-5), giant rotation by -g'b, sum, one rescale.  Depth 1."""
    W = len(taps)
    b, giants = fir_rot_schedule(W)
    babies = [x] + [r[0] for r in baby_steps(ev, [x], [-s for s in range(1, min(b, W))], hoist)]
    inners = [ev.lincomb_scalar([babies[s] for s in ss], [taps[gp * b + s] for s in ss]) for gp, ss in giants]
    acc = None
    for (gp, ss), inner in zip(giants, inners):
        if gp:
            inner = ev.rotate(inner, -gp * b)
        acc = inner if acc is None else ev.add(acc, inner)
    return ev.rescale(acc)


def k7_taylor_phase(ev, If, Qf, order):
    """K7: y[t] = Q_f[t] I_f[t-1] - I_f[t] Q_f[t-1]; first order y,
    third order y x^2 - y^3/3 (literal polynomial, reading #2); t = 1..F-1."""
    if order not in (1, 3):
        raise ValueError(f"taylor order must be 1 or 3, got {order}")
    T = range(1, len(If))
    ty = [ev.tensor_sum([(Qf[t], If[t - 1])]) for t in T]
    ty2 = [ev.tensor_sum([(If[t], Qf[t - 1])]) for t in T]
    y = ev.relin_rescale_all([ev.sub(a, b) for a, b in zip(ty, ty2)])
    if order == 1:
        return y
    x = ev.relin_rescale_all([ev.tensor_sum([(If[t], If[t - 1]), (Qf[t], Qf[t - 1])]) for t in T])
    x2 = ev.square_rescale_all(x)
    y2 = ev.square_rescale_all(y)
    yt = [ev.rescale(v) for v in [ev.lincomb_scalar([v], [-1.0 / 3.0]) for v in y]]
    yd = [ev.drop_to(v, w.level) for v, w in zip(y, x2)]
    yx2 = ev.relin_rescale_all([ev.tensor_sum([(v, w)]) for v, w in zip(yd, x2)])
    y3 = ev.relin_rescale_all([ev.tensor_sum([(v, w)]) for v, w in zip(y2, yt)])
    return [ev.add(a, b) for a, b in zip(yx2, y3)]


def vp_band_power(ev, ys, bins):
    """VP+ (P:279-288): X[k] = sum_t c_{k,t} y[t] (+ j s_{k,t}), P_k = |X[k]|^2."""
    Fp = len(ys)
    coefs = [dsp.narrowband_dft_coefs(Fp, int(k)) for k in bins]
    xr = [ev.lincomb_scalar(ys, c) for c, _ in coefs]
    xi = [ev.lincomb_scalar(ys, s) for _, s in coefs]
    xr = [ev.rescale(x) for x in xr]
    xi = [ev.rescale(x) for x in xi]
    return ev.relin_rescale_all([ev.tensor_sum([(a, a), (b, b)]) for a, b in zip(xr, xi)])


def vp_weighted_average(ev, Pk, bins, fs, Fp):
    """VP+ sharpen and weighted frequency average:
    S_k = P_k^2 (HMult + relin + rescale), N_f = sum_k f_k S_k, D_f = sum_k S_k with
    f_k = k fs / Fp Hz as scalar constants (every PMult rescaled); the client reads
    BPM = 60 N_f / D_f.  Op-major: both sums, then both rescales."""
    S = ev.square_rescale_all(Pk)
    f = [float(k) * fs / Fp for k in bins]
    lin = [ev.lincomb_scalar(S, f), ev.lincomb_scalar(S, [1.0] * len(S))]
    return [ev.rescale(x) for x in lin]


def vitals_v2(ev, re_list, im_list, taps_by_band, cfg):
    """Chain V2: K4 -> K5 -> K7 -> narrowband DFT -> |X|^2 per band;
    returns {band index: [P_k ciphertexts]} (sharpen/average on the client, reading #4),
    or with cfg.vp_plus {band index: [N_f, D_f]} (VP+ in the cloud, the full-depth chain)."""
    set_merge(ev, cfg)
    I, Q = [], []
    for s, e in chunks(len(re_list), cfg.frame_batch):
        Ib, Qb = k4_soft_iq(ev, re_list[s:e], im_list[s:e], cfg)
        I += Ib
        Q += Qb
    out = {}
    for bi, taps in enumerate(taps_by_band):
        If = k5_fir(ev, I, taps)
        Qf = k5_fir(ev, Q, taps)
        ys = k7_taylor_phase(ev, If, Qf, cfg.taylor_order)
        bins = dsp.band_bins(len(ys), cfg.fs, cfg.bands[bi])
        out[bi] = vp_band_power(ev, ys, bins)
        if cfg.vp_plus:
            out[bi] = vp_weighted_average(ev, out[bi], bins, cfg.fs, len(ys))
    return out


# ------------------------------------------------------------------ key sets

def rotsum_steps(count: int, stride: int):
    out, s, c = [], stride, 1
    while c < count:
        out.append(s)
        s *= 2
        c *= 2
    return out


def required_rotations(chain: str, cfg: ChainCfg, n_ring: int):
    """Rotation amounts (normalised to [0, N/2)) a chain needs, plus the
    conjugation key id orc.CONJ where K1 runs on complex slots (reading R28)."""
    half = n_ring // 2
    ks = set()
    extra = {orc.CONJ} if cplx_of(cfg) and chain in ("gesture_frame", "gesture", "gesture_features") else set()
    if extra and getattr(cfg, "k1_conj_fuse", 0):
        extra.add(orc.CONJ_PROD)
    if chain == "k5_fir_rot":
        W = max(cfg.n_taps) if getattr(cfg, "n_taps", None) else 0
        b, giants = fir_rot_schedule(W) if W else (1, [])
        ks |= {-s for s in range(1, min(b, W))} | {-gp * b for gp, _ in giants if gp}
    if chain in ("k2_soft_attention", "vitals_v1", "k4_soft_iq", "vitals_v2"):
        ks |= set(rotsum_steps(cfg.R, 1))
    if chain in ("k4_soft_iq", "vitals_v2") and cfg.iq_pack:
        log2_exact(cfg.R, "R (iq_pack)")
        for j in range(cfg.iq_pack):
            ks |= {cfg.R << j, -(cfg.R << j)}
        if cfg.hoist:
            ks |= {m * cfg.R for m in range(1, 1 << cfg.iq_pack)}
    L = lanes_of(cfg)

    def rotsum_keys(count, stride):  # + the double-hoisted levels' strides (R27 / R30)
        if not dh(cfg):
            return set(rotsum_steps(count, stride))
        out, st, c = set(), stride, count
        for a in rotsum_levels(count, rotsum_inner(cfg), bool(getattr(cfg, "rotsum_hoist_all", 0))):
            out |= {j * st for j in range(1, a)}
            st *= a
            c //= a
        return out | set(rotsum_steps(c, st))
        return out

    if chain in ("k3_doppler_dft", "gesture_frame", "gesture", "gesture_features"):
        b, giants = k3_schedule(cfg)
        ks |= {s * L for s in range(1, b)}
        ks |= {G * L for _, G, _ in giants if G != 0}
    if chain in ("k2_doppler_soft_power", "gesture_frame", "gesture", "gesture_features"):
        ks |= rotsum_keys(cfg.n_slots // cfg.D, cfg.D * L)
    if chain in ("gesture_fc", "gesture", "fc_forward"):
        ks |= rotsum_keys(L, 1)
        dims = cfg.fc_dims
        for layer in range(len(dims) - 1):
            h = dims[layer + 1]
            b, giants = fc_schedule(h, getattr(cfg, "fc_baby", 0))
            ks |= {s * L for s in range(1, min(b, h))}
            ks |= {G * L for _, G, _ in giants if G != 0}
            ks |= rotsum_keys(dims[layer] // h, h * L)
    return sorted(({k % half for k in ks} - {0}) | extra)
