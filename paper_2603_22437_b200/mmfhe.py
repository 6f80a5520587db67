"""Thin ctypes binding of include/mmfhe.h (argument marshalling only).

Every computation happens in libmmfhe.so's CUDA kernels; there is no CPU
fallback: if the library is missing this module raises at import/load time.
Buffers are numpy uint64 arrays (host) or torch int64/uint64 CUDA tensors
(device, passed by data_ptr()).  Names follow the C-ABI.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MMFHE_LIB selects another build of the same library (tools/build_variant.py experiments)
LIB_PATH = os.environ.get("MMFHE_LIB") or os.path.join(_HERE, "lib", "libmmfhe.so")

FORM_COEFF, FORM_EVAL = 0, 1

STATUS = {
    0: "OK", 1: "E_INVALID_ARG", 2: "E_PARAMS", 3: "E_DEPTH", 4: "E_MISSING_KEY", 5: "E_LAYOUT",
    6: "E_SCALE", 7: "E_SHAPE", 8: "E_CUDA", 9: "E_OOM", 10: "E_NCCL", 11: "E_FORMAT", 12: "E_MISSING_PLAIN",
}


class MmfheError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Params(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n_q", ctypes.c_uint32), ("q", ctypes.POINTER(ctypes.c_uint64)),
                ("n_p", ctypes.c_uint32), ("p", ctypes.POINTER(ctypes.c_uint64)), ("alpha", ctypes.c_uint32),
                ("scale_bits", ctypes.c_uint32), ("security", ctypes.c_uint32)]


class CT(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("level", ctypes.c_uint32), ("n_slots", ctypes.c_uint32),
                ("form", ctypes.c_uint32), ("scale", ctypes.c_double), ("data", ctypes.c_void_p),
                ("on_device", ctypes.c_int32), ("n_polys", ctypes.c_uint32)]


class ChainCfg(ctypes.Structure):
    _fields_ = [("R", ctypes.c_uint32), ("D", ctypes.c_uint32), ("A", ctypes.c_uint32), ("F", ctypes.c_uint32),
                ("gamma", ctypes.c_uint32), ("p_phi", ctypes.c_uint32), ("taylor_order", ctypes.c_uint32),
                ("n_slots", ctypes.c_uint32), ("bsgs_baby", ctypes.c_uint32), ("hoist", ctypes.c_uint32),
                ("frame_batch", ctypes.c_uint32), ("fc_dims", ctypes.c_uint32 * 4), ("notch_width", ctypes.c_uint32), ("n_bands", ctypes.c_uint32),
                ("n_taps", ctypes.c_uint32 * 4), ("n_bins", ctypes.c_uint32 * 4),
                ("bins", (ctypes.c_uint32 * 64) * 4), ("fs", ctypes.c_double), ("vp_plus", ctypes.c_uint32),
                ("iq_pack", ctypes.c_uint32), ("lanes", ctypes.c_uint32), ("fc_baby", ctypes.c_uint32),
                ("cplx", ctypes.c_uint32), ("bsgs_aligned", ctypes.c_uint32), ("rotsum_inner", ctypes.c_uint32),
                ("rotsum_hoist_all", ctypes.c_uint32), ("ks_merge", ctypes.c_uint32),
                ("k1_conj_fuse", ctypes.c_uint32), ("sessions", ctypes.c_uint32)]

# Key id of the conjugation automorphism (include/mmfhe.h MMFHE_STEP_CONJ, DESIGN R28)
STEP_CONJ = -(1 << 31)
STEP_CONJ_PROD = STEP_CONJ + 1  # the conjugate-product key (MMFHE_STEP_CONJ_PROD, DESIGN R32)


def chain_cfg(R=0, D=0, A=0, F=0, gamma=1, p_phi=1, taylor_order=1, n_slots=0, bsgs_baby=0,
              fc_dims=(0, 0, 0, 0), notch_width=1, bands_bins=(), n_taps=(), fs=0.0, frame_batch=0,
              hoist=0, vp_plus=0, iq_pack=0, lanes=1, fc_baby=0, cplx=0, bsgs_aligned=0,
              rotsum_inner=0, rotsum_hoist_all=0, ks_merge=0, k1_conj_fuse=0, sessions=0) -> ChainCfg:
    c = ChainCfg()
    c.R, c.D, c.A, c.F = R, D, A, F
    c.gamma, c.p_phi, c.taylor_order, c.n_slots, c.bsgs_baby = gamma, p_phi, taylor_order, n_slots, bsgs_baby
    c.frame_batch, c.hoist = frame_batch, hoist
    for i, v in enumerate(fc_dims):
        c.fc_dims[i] = int(v)
    c.notch_width = notch_width
    c.n_bands = len(bands_bins)
    for b, bins in enumerate(bands_bins):
        c.n_bins[b] = len(bins)
        for i, k in enumerate(bins):
            c.bins[b][i] = int(k)
    for b, t in enumerate(n_taps):
        c.n_taps[b] = int(t)
    c.fs = float(fs)
    c.vp_plus = int(vp_plus)
    c.iq_pack = int(iq_pack)
    c.lanes = int(lanes)
    c.fc_baby = int(fc_baby)
    c.cplx = int(cplx)
    c.bsgs_aligned = int(bsgs_aligned)
    c.rotsum_inner = int(rotsum_inner)
    c.rotsum_hoist_all = int(rotsum_hoist_all)
    c.ks_merge = int(ks_merge)
    c.k1_conj_fuse = int(k1_conj_fuse)
    c.sessions = int(sessions)
    return c


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -m paper_2603_22437_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, V, S, U32, U64, I32 = (ctypes.POINTER, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32,
                                  ctypes.c_uint64, ctypes.c_int32)
        CTP = P(CT)
        sig = {
            "mmfhe_ctx_create": [P(Params), ctypes.c_int, V, P(V)],
            "mmfhe_ctx_destroy": [V],
            "mmfhe_ctx_memory": [V, P(S)],
            "mmfhe_launch_count": [V, P(U64)],
            "mmfhe_chain_required_rotations": [V, ctypes.c_char_p, P(ChainCfg), P(I32), S, P(S)],
            "mmfhe_load_relin_key": [V, V, S, ctypes.c_int],
            "mmfhe_load_galois_key": [V, I32, V, S, ctypes.c_int],
            "mmfhe_load_plain": [V, ctypes.c_char_p, CTP],
            "mmfhe_load_plain_pq": [V, ctypes.c_char_p, CTP],
            "mmfhe_encode_plain": [V, ctypes.c_char_p, P(ctypes.c_double), S, U32, ctypes.c_double],
            "mmfhe_prepare_chain": [V, ctypes.c_char_p, P(ChainCfg), U32, V, V, V],
            "mmfhe_load_scalars": [V, ctypes.c_char_p, P(ctypes.c_double), S],
            "mmfhe_chain_plan": [V, ctypes.c_char_p, P(ChainCfg), U32, S, P(U32), S, P(S)],
            "mmfhe_eval_chain": [V, ctypes.c_char_p, P(ChainCfg), CTP, S, CTP, S, P(S)],
            "mmfhe_eval_chain_async": [V, ctypes.c_char_p, P(ChainCfg), CTP, S, CTP, S, P(S)],
            "mmfhe_ctx_sync": [V],
            "mmfhe_sum_partials": [V, CTP, S, CTP],
            "mmfhe_ntt": [V, V, U32, P(U32)],
            "mmfhe_intt": [V, V, U32, P(U32)],
            "mmfhe_hadd": [V, CTP, CTP, CTP],
            "mmfhe_hsub": [V, CTP, CTP, CTP],
            "mmfhe_pmult": [V, CTP, ctypes.c_char_p, CTP],
            "mmfhe_hmult": [V, CTP, CTP, CTP],
            "mmfhe_relin": [V, CTP, CTP],
            "mmfhe_hrot": [V, CTP, I32, CTP],
            "mmfhe_hrot_hoisted": [V, CTP, P(I32), S, CTP],
            "mmfhe_hrot_hoisted_pq": [V, CTP, P(I32), S, CTP],
            "mmfhe_rescale": [V, CTP, CTP],
            "mmfhe_keyswitch": [V, CTP, I32, ctypes.c_int, CTP],
            "mmfhe_mod_switch": [V, CTP, U32, CTP],
            "mmfhe_hrot_batch": [V, CTP, S, I32, CTP],
            "mmfhe_hmult_batch": [V, CTP, CTP, S, CTP],
            "mmfhe_trace_get": [V, ctypes.c_char_p, S, P(S)],
            "mmfhe_trace_clear": [V],
            "mmfhe_trace_enable": [V, ctypes.c_int],
            "mmfhe_graph_enable": [V, ctypes.c_int],
            "mmfhe_graph_stats": [V, P(S), P(ctypes.c_uint64)],
            "mmfhe_profile_enable": [V, ctypes.c_int],
            "mmfhe_profile_get": [V, ctypes.c_char_p, S, P(S)],
            "mmfhe_microbench": [V, ctypes.c_int, P(ctypes.c_double)],
            "mmfhe_params_digest": [V, P(U64)],
            "mmfhe_serialize_ct": [V, CTP, V, S, P(S)],
            "mmfhe_deserialize_ct": [V, V, S, CTP],
            "mmfhe_serialize_key": [V, ctypes.c_int, I32, V, S, ctypes.c_int, V, S, P(S)],
            "mmfhe_load_key_serialized": [V, V, S],
            "mmfhe_client_keygen": [V, U64, P(I32), S, ctypes.c_int, V, V, V, ctypes.c_int],
            "mmfhe_client_encrypt": [V, V, ctypes.c_int, CTP, S, U64, U32, CTP],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.mmfhe_last_error.argtypes = [V]
        L.mmfhe_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


# symbols the header declares (checked by the CPU test suite)
EXPORTED = [
    "mmfhe_ctx_create", "mmfhe_ctx_destroy", "mmfhe_last_error", "mmfhe_ctx_memory", "mmfhe_launch_count",
    "mmfhe_chain_required_rotations", "mmfhe_load_relin_key", "mmfhe_load_galois_key", "mmfhe_load_plain",
    "mmfhe_encode_plain", "mmfhe_prepare_chain", "mmfhe_load_scalars", "mmfhe_chain_plan", "mmfhe_eval_chain",
    "mmfhe_sum_partials", "mmfhe_ntt", "mmfhe_intt", "mmfhe_hadd", "mmfhe_hsub", "mmfhe_pmult", "mmfhe_hmult",
    "mmfhe_relin", "mmfhe_hrot", "mmfhe_hrot_hoisted", "mmfhe_hrot_hoisted_pq", "mmfhe_rescale", "mmfhe_keyswitch", "mmfhe_mod_switch", "mmfhe_hrot_batch",
    "mmfhe_hmult_batch", "mmfhe_trace_get", "mmfhe_trace_clear", "mmfhe_trace_enable", "mmfhe_profile_enable",
    "mmfhe_profile_get", "mmfhe_microbench", "mmfhe_graph_enable", "mmfhe_graph_stats", "mmfhe_eval_chain_async",
    "mmfhe_ctx_sync", "mmfhe_params_digest", "mmfhe_serialize_ct", "mmfhe_deserialize_ct", "mmfhe_serialize_key",
    "mmfhe_load_key_serialized", "mmfhe_load_plain_pq", "mmfhe_client_keygen", "mmfhe_client_encrypt",
]

SER_CT, SER_RELIN_KEY, SER_GALOIS_KEY = 0, 1, 2


def _u64_array(vals):
    a = (ctypes.c_uint64 * len(vals))()
    for i, v in enumerate(vals):
        a[i] = int(v)
    return a


def _ptr(buf):
    """(address, on_device) of a numpy array or torch tensor."""
    if isinstance(buf, np.ndarray):
        assert buf.dtype == np.uint64 and buf.flags["C_CONTIGUOUS"], "host buffers: C-contiguous uint64"
        return buf.ctypes.data, 0
    if hasattr(buf, "data_ptr"):
        assert buf.is_contiguous() and buf.element_size() == 8, "device buffers: contiguous 64-bit tensor"
        return buf.data_ptr(), 1 if buf.is_cuda else 0
    raise TypeError(f"unsupported buffer {type(buf)}")


@dataclass
class Ct:
    """A ciphertext/plaintext buffer + metadata as seen by the C-ABI."""
    data: object             # numpy uint64 (host) or torch 64-bit tensor (device)
    level: int
    scale: float
    n_slots: int
    log_n: int
    form: int = FORM_COEFF
    n_polys: int = 2

    def struct(self) -> CT:
        addr, dev = _ptr(self.data)
        return CT(self.log_n, self.level, self.n_slots, self.form, float(self.scale), addr, dev, self.n_polys)


class CtArray:
    """A marshalled mmfhe_ct[] built once from a list of Ct (the buffers must stay alive);
    passing it to eval_chain avoids rebuilding thousands of structs per call."""

    def __init__(self, cts):
        self.cts = list(cts)
        self.arr = (CT * len(self.cts))(*[c.struct() for c in self.cts])

    def __len__(self):
        return len(self.cts)

    def sync_back(self):
        for c, s in zip(self.cts, self.arr):
            c.level, c.scale, c.n_slots = s.level, s.scale, s.n_slots


class Context:
    def __init__(self, log_n, q, p, alpha, scale_bits, device=0, stream=None):
        self._lib = lib()
        self.log_n, self.n = log_n, 1 << log_n
        self.q, self.p = [int(x) for x in q], [int(x) for x in p]
        self.alpha, self.scale_bits = alpha, scale_bits
        self._qa, self._pa = _u64_array(self.q), _u64_array(self.p)
        prm = Params(log_n, len(self.q), self._qa, len(self.p), self._pa, alpha, scale_bits, 128)
        h = ctypes.c_void_p()
        st = self._lib.mmfhe_ctx_create(ctypes.byref(prm), device, ctypes.c_void_p(stream or 0), ctypes.byref(h))
        if st:
            raise MmfheError(st, self._lib.mmfhe_last_error(None).decode())
        self.h = h

    @classmethod
    def from_params(cls, P, device=0, stream=None):
        return cls(P.log_n, P.q, P.p, P.alpha, P.scale_bits, device, stream)

    def close(self):
        if getattr(self, "h", None):
            self._lib.mmfhe_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st:
            raise MmfheError(st, self._lib.mmfhe_last_error(self.h).decode())

    # ---- keys / operands
    def load_relin_key(self, words):
        addr, dev = _ptr(words)
        self._check(self._lib.mmfhe_load_relin_key(self.h, addr, _numel(words), dev))

    def load_galois_key(self, step, words):
        addr, dev = _ptr(words)
        self._check(self._lib.mmfhe_load_galois_key(self.h, int(step), addr, _numel(words), dev))

    def load_plain(self, name, residues, level, scale):
        """Import a coefficient-form plaintext; a name ending in ".pq" is over Q_level u P
        (residues [level+1+K][N], mmfhe_load_plain_pq; stored under that name)."""
        ct = Ct(residues, level, scale, 0, self.log_n, FORM_COEFF, 1)
        s = ct.struct()
        if name.endswith(".pq"):
            self._check(self._lib.mmfhe_load_plain_pq(self.h, name[:-3].encode(), ctypes.byref(s)))
        else:
            self._check(self._lib.mmfhe_load_plain(self.h, name.encode(), ctypes.byref(s)))

    def encode_plain(self, name, values, level, scale):
        v = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self._lib.mmfhe_encode_plain(self.h, name.encode(),
                                                 v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                 len(v), level, float(scale)))

    def load_scalars(self, name, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self._lib.mmfhe_load_scalars(self.h, name.encode(),
                                                 v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(v)))

    def prepare_chain(self, chain, cfg, in_level, fc_w=None, fc_b=None, taps=None):
        keep = []

        def arr_list(mats):
            if mats is None:
                return None
            ptrs = (ctypes.c_void_p * len(mats))()
            for i, m in enumerate(mats):
                a = np.ascontiguousarray(m, dtype=np.float64)
                keep.append(a)
                ptrs[i] = a.ctypes.data
            keep.append(ptrs)
            return ptrs

        self._check(self._lib.mmfhe_prepare_chain(self.h, chain.encode(), ctypes.byref(cfg), in_level,
                                                  arr_list(fc_w), arr_list(fc_b), arr_list(taps)))

    def required_rotations(self, chain, cfg):
        n = ctypes.c_size_t()
        self._check(self._lib.mmfhe_chain_required_rotations(self.h, chain.encode(), ctypes.byref(cfg), None, 0,
                                                             ctypes.byref(n)))
        buf = (ctypes.c_int32 * max(n.value, 1))()
        self._check(self._lib.mmfhe_chain_required_rotations(self.h, chain.encode(), ctypes.byref(cfg), buf,
                                                             n.value, ctypes.byref(n)))
        return [buf[i] for i in range(n.value)]

    def chain_plan(self, chain, cfg, in_level, n_in):
        n = ctypes.c_size_t()
        buf = (ctypes.c_uint32 * 1024)()
        self._check(self._lib.mmfhe_chain_plan(self.h, chain.encode(), ctypes.byref(cfg), in_level, n_in, buf, 1024,
                                               ctypes.byref(n)))
        return [buf[i] for i in range(n.value)]

    def eval_chain(self, chain, cfg, ins, outs):
        """ins / outs: lists of Ct, or CtArray (pre-marshalled, reused across calls)."""
        arr_in = ins if isinstance(ins, CtArray) else CtArray(ins)
        arr_out = outs if isinstance(outs, CtArray) else CtArray(outs)
        n = ctypes.c_size_t()
        self._check(self._lib.mmfhe_eval_chain(self.h, chain.encode(), ctypes.byref(cfg), arr_in.arr, len(arr_in),
                                               arr_out.arr, len(arr_out), ctypes.byref(n)))
        arr_out.sync_back()
        return n.value

    def eval_chain_async(self, chain, cfg, ins, outs):
        """Non-blocking eval_chain for host (pinned) buffers: upload of call i+1 overlaps
        the compute of call i.  Keep the buffers alive; read outputs after sync()."""
        arr_in = ins if isinstance(ins, CtArray) else CtArray(ins)
        arr_out = outs if isinstance(outs, CtArray) else CtArray(outs)
        n = ctypes.c_size_t()
        self._check(self._lib.mmfhe_eval_chain_async(self.h, chain.encode(), ctypes.byref(cfg), arr_in.arr,
                                                     len(arr_in), arr_out.arr, len(arr_out), ctypes.byref(n)))
        arr_out.sync_back()
        return n.value

    def sync(self):
        """Wait for all work enqueued on this context (copy and compute streams)."""
        self._check(self._lib.mmfhe_ctx_sync(self.h))

    # ---- primitives
    def ntt(self, rows, prime_idx, inverse=False):
        addr, dev = _ptr(rows)
        assert dev, "NTT works on device buffers"
        idx = (ctypes.c_uint32 * len(prime_idx))(*[int(i) for i in prime_idx])
        f = self._lib.mmfhe_intt if inverse else self._lib.mmfhe_ntt
        self._check(f(self.h, addr, len(prime_idx), idx))

    def _unary(self, fname, a: Ct, out: Ct, *extra):
        sa, so = a.struct(), out.struct()
        self._check(getattr(self._lib, fname)(self.h, ctypes.byref(sa), *extra, ctypes.byref(so)))
        out.level, out.scale, out.n_slots, out.n_polys = so.level, so.scale, so.n_slots, so.n_polys
        return out

    def _binary(self, fname, a: Ct, b: Ct, out: Ct):
        sa, sb, so = a.struct(), b.struct(), out.struct()
        self._check(getattr(self._lib, fname)(self.h, ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(so)))
        out.level, out.scale, out.n_slots, out.n_polys = so.level, so.scale, so.n_slots, so.n_polys
        return out

    def hadd(self, a, b, out):
        return self._binary("mmfhe_hadd", a, b, out)

    def hsub(self, a, b, out):
        return self._binary("mmfhe_hsub", a, b, out)

    def hmult(self, a, b, out):
        return self._binary("mmfhe_hmult", a, b, out)

    def pmult(self, a, name, out):
        return self._unary("mmfhe_pmult", a, out, name.encode())

    def relin(self, a3, out):
        return self._unary("mmfhe_relin", a3, out)

    def hrot(self, a, step, out):
        return self._unary("mmfhe_hrot", a, out, int(step))

    def hrot_hoisted(self, a, steps, outs):
        sa = a.struct()
        st = (ctypes.c_int32 * len(steps))(*[int(s) for s in steps])
        o = (CT * len(outs))(*[c.struct() for c in outs])
        self._check(self._lib.mmfhe_hrot_hoisted(self.h, ctypes.byref(sa), st, len(steps), o))
        for c, s in zip(outs, o):
            c.level, c.scale, c.n_slots = s.level, s.scale, s.n_slots
        return outs

    def hrot_hoisted_pq(self, a, steps, outs):
        """Double-hoisted baby steps: outs[i] <- PQ ciphertext of step i (data: 2 (level+1+K) N words,
        Q rows of poly 0 / poly 1, then P rows of poly 0 / poly 1)."""
        sa = a.struct()
        st = (ctypes.c_int32 * len(steps))(*[int(s) for s in steps])
        o = (CT * len(outs))(*[c.struct() for c in outs])
        self._check(self._lib.mmfhe_hrot_hoisted_pq(self.h, ctypes.byref(sa), st, len(steps), o))
        for c, s in zip(outs, o):
            c.level, c.scale, c.n_slots = s.level, s.scale, s.n_slots
        return outs

    def rescale(self, a, out):
        return self._unary("mmfhe_rescale", a, out)

    def mod_switch(self, a, level, out):
        return self._unary("mmfhe_mod_switch", a, out, int(level))

    def keyswitch(self, x, out, step=0, use_relin=True):
        return self._unary("mmfhe_keyswitch", x, out, int(step), 1 if use_relin else 0)

    def sum_partials(self, parts, out):
        arr = (CT * len(parts))(*[c.struct() for c in parts])
        so = out.struct()
        self._check(self._lib.mmfhe_sum_partials(self.h, arr, len(parts), ctypes.byref(so)))
        out.level, out.scale = so.level, so.scale
        return out

    def hrot_batch(self, cts, step, outs):
        a = (CT * len(cts))(*[c.struct() for c in cts])
        o = (CT * len(outs))(*[c.struct() for c in outs])
        self._check(self._lib.mmfhe_hrot_batch(self.h, a, len(cts), int(step), o))

    def hmult_batch(self, xs, ys, outs):
        a = (CT * len(xs))(*[c.struct() for c in xs])
        b = (CT * len(ys))(*[c.struct() for c in ys])
        o = (CT * len(outs))(*[c.struct() for c in outs])
        self._check(self._lib.mmfhe_hmult_batch(self.h, a, b, len(xs), o))

    # ---- trace / counters
    def trace(self):
        n = ctypes.c_size_t()
        self._check(self._lib.mmfhe_trace_get(self.h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        self._check(self._lib.mmfhe_trace_get(self.h, buf, n.value + 1, ctypes.byref(n)))
        return [tuple(_parse_trace(line)) for line in buf.value.decode().splitlines()]

    def trace_clear(self):
        self._check(self._lib.mmfhe_trace_clear(self.h))

    def trace_enable(self, on=True):
        self._check(self._lib.mmfhe_trace_enable(self.h, 1 if on else 0))

    def graph_enable(self, on=True):
        """CUDA-graph replay of repeated device-resident eval_chain calls (default on)."""
        self._check(self._lib.mmfhe_graph_enable(self.h, 1 if on else 0))

    def graph_stats(self):
        """(captured graphs held, graph replays so far)."""
        n, r = ctypes.c_size_t(), ctypes.c_uint64()
        self._check(self._lib.mmfhe_graph_stats(self.h, ctypes.byref(n), ctypes.byref(r)))
        return n.value, r.value

    def profile_enable(self, on=True):
        self._check(self._lib.mmfhe_profile_enable(self.h, 1 if on else 0))

    def profile(self):
        """{kernel: (launches, total_ms, algorithmic_bytes)} since the last call (resets)."""
        n = ctypes.c_size_t()
        buf = ctypes.create_string_buffer(1 << 16)
        self._check(self._lib.mmfhe_profile_get(self.h, buf, 1 << 16, ctypes.byref(n)))
        out = {}
        for line in buf.value.decode().splitlines():
            k, c, ms, b, ops = line.split()
            out[k] = (int(c), float(ms), float(b), float(ops))
        return out

    # ---- serialisation (include/mmfhe.h documents the blob layout)
    def params_digest(self):
        d = ctypes.c_uint64()
        self._check(self._lib.mmfhe_params_digest(self.h, ctypes.byref(d)))
        return int(d.value)

    def serialize_ct(self, ct) -> bytes:
        s = ct.struct()
        n = ctypes.c_size_t()
        self._check(self._lib.mmfhe_serialize_ct(self.h, ctypes.byref(s), None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        self._check(self._lib.mmfhe_serialize_ct(self.h, ctypes.byref(s), buf, n.value, ctypes.byref(n)))
        return buf.raw[: n.value]

    def deserialize_ct(self, blob: bytes, out):
        s = out.struct()
        self._check(self._lib.mmfhe_deserialize_ct(self.h, blob, len(blob), ctypes.byref(s)))
        out.level, out.scale, out.n_slots, out.n_polys, out.form = s.level, s.scale, s.n_slots, s.n_polys, s.form
        return out

    def serialize_key(self, kind, step, words) -> bytes:
        addr, dev = _ptr(words)
        n = ctypes.c_size_t()
        self._check(self._lib.mmfhe_serialize_key(self.h, kind, int(step), addr, _numel(words), dev, None, 0,
                                                  ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        self._check(self._lib.mmfhe_serialize_key(self.h, kind, int(step), addr, _numel(words), dev, buf, n.value,
                                                  ctypes.byref(n)))
        return buf.raw[: n.value]

    def load_key_serialized(self, blob: bytes):
        self._check(self._lib.mmfhe_load_key_serialized(self.h, blob, len(blob)))

    # ---- the trusted client on the GPU (include/mmfhe.h: never used by the cloud side)
    def client_keygen(self, seed, steps=(), relin=True, pk=None, rlk=None, gk=None):
        """pk [2][L+1][N], rlk and gk[i] [dnum][2][L+1+K][N] into the given buffers (numpy or
        CUDA tensors, all on one side) or new numpy arrays; returns (pk, rlk, gk)."""
        L1, K1 = len(self.q), len(self.q) + len(self.p)
        dn = -(-L1 // self.alpha)
        if pk is None:
            pk = np.empty((2, L1, self.n), dtype=np.uint64)
            rlk = np.empty((dn, 2, K1, self.n), dtype=np.uint64) if relin else None
            gk = np.empty((len(steps), dn, 2, K1, self.n), dtype=np.uint64) if steps else None
        st = (ctypes.c_int32 * max(len(steps), 1))(*[int(s) for s in steps])
        addr, dev = _ptr(pk)
        r_addr = _ptr(rlk)[0] if rlk is not None else None
        g_addr = _ptr(gk)[0] if gk is not None else None
        self._check(self._lib.mmfhe_client_keygen(self.h, int(seed), st, len(steps), 1 if relin else 0, addr,
                                                  r_addr, g_addr, dev))
        return pk, rlk, gk

    def client_encrypt(self, pk, pts, seed, first_index, outs):
        """outs[i] = Enc(pts[i]) with the encryption streams of index first_index + i."""
        addr, dev = _ptr(pk)
        ai, ao = CtArray(pts), CtArray(outs)
        self._check(self._lib.mmfhe_client_encrypt(self.h, addr, dev, ai.arr, len(ai), int(seed), int(first_index),
                                                   ao.arr))
        ao.sync_back()
        return outs

    def microbench(self, kind):
        """Whole-GPU ops/s of one register-resident op: 0 CT butterfly, 1 GS butterfly,
        2 64x64->128 MAC, 3 Shoup modular product."""
        v = ctypes.c_double()
        self._check(self._lib.mmfhe_microbench(self.h, int(kind), ctypes.byref(v)))
        return v.value

    def launch_count(self):
        c = ctypes.c_uint64()
        self._check(self._lib.mmfhe_launch_count(self.h, ctypes.byref(c)))
        return c.value

    def memory(self):
        c = ctypes.c_size_t()
        self._check(self._lib.mmfhe_ctx_memory(self.h, ctypes.byref(c)))
        return c.value


def _parse_trace(line):
    parts = line.split(" ")
    op, level = parts[0], int(parts[1])
    arg = parts[2] if len(parts) > 2 else ""
    return op, level, arg


def _numel(buf):
    if isinstance(buf, np.ndarray):
        return buf.size
    return buf.numel()
