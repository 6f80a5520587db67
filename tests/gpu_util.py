"""Helpers shared by the GPU parity tests: move oracle objects into a GPU
context through the C-ABI binding and compare residues."""
from __future__ import annotations

import numpy as np

from synth import prng


def dev_tensor(arr: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint64).view(np.int64)).to("cuda:0")


def host(t) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def ct_in(m, P, ct, device=True):
    """oracle Ct -> binding Ct (coefficient form)."""
    data = np.ascontiguousarray(np.stack(ct.c))
    return m.Ct(dev_tensor(data) if device else data, ct.level, ct.scale, ct.n_slots, P.log_n,
                m.FORM_COEFF, len(ct.c))


def ct_out(m, P, level, npolys=2, device=True):
    import torch
    shape = (npolys, level + 1, P.n)
    data = torch.empty(shape, dtype=torch.int64, device="cuda:0") if device else np.empty(shape, dtype=np.uint64)
    return m.Ct(data, level, 0.0, 0, P.log_n, m.FORM_COEFF, npolys)


def residues(x) -> np.ndarray:
    return host(x.data) if not isinstance(x.data, np.ndarray) else x.data


def make_ctx(m, P, keys=None, book=None, scalars=None):
    ctx = m.Context.from_params(P)
    if keys is not None:
        if keys.rlk is not None:
            ctx.load_relin_key(keys.rlk)
        for k, evk in keys.gk.items():
            ctx.load_galois_key(k, evk)
    if book is not None:
        for (name, level), (res, sc, _) in book.entries.items():
            ctx.load_plain(name, np.ascontiguousarray(res), level, sc)
    for name, vals in (scalars or {}).items():
        ctx.load_scalars(name, vals)
    return ctx


def uniform_poly(P, level, seed, sid, npolys=1):
    """Uniform residues [npolys][level+1][N] (ciphertext-distributed)."""
    out = np.empty((npolys, level + 1, P.n), dtype=np.uint64)
    for p in range(npolys):
        for i in range(level + 1):
            out[p, i] = prng.uniform_mod(seed, sid + p, P.n, P.q[i], offset=i * P.n)
    return out
