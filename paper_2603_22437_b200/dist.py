"""Multi-GPU plumbing for the mmFHE hot path.

Units are independent (sessions, frames); the method's only exchange step is the
cross-frame homomorphic sum ("accumulate across frames via addition",
P:943) when one session's frames are spread over GPUs: each rank evaluates the
frame kernels on its frame shard and sums them locally (chain
``gesture_features``), the per-rank partial ciphertexts are all-gathered over
NCCL/NVLink, and the modular sum of the gathered parts runs in the library
(``mmfhe_sum_partials``) before the FC head.

torch.distributed only moves bytes (NCCL on GPUs, gloo in the CPU tests); no
arithmetic of the method happens here.
"""
from __future__ import annotations


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) share of n units for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def owner(unit: int, world: int) -> int:
    """Rank that finishes unit (session) `unit` after the exchange (round-robin)."""
    return unit % world


def allgather_partials(local, group=None):
    """[k, ...] 64-bit tensor of per-rank partial ciphertexts -> [world, k, ...] on every
    rank (rank order).  A no-op stack when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    local = local.contiguous()
    if not (dist.is_available() and dist.is_initialized()):
        return local.unsqueeze(0)
    world = dist.get_world_size(group)
    k = local.shape[0]
    if dist.get_backend(group) == "gloo" and local.is_cuda:
        # gloo (multi-process checks on one GPU) gathers host tensors; NCCL gathers in HBM
        parts = [torch.empty_like(local, device="cpu") for _ in range(world)]
        dist.all_gather(parts, local.cpu(), group=group)
        return torch.stack(parts).to(local.device)
    out = torch.empty((world * k,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)  # rank-major concatenation
    return out.view((world, k) + tuple(local.shape[1:]))


def sessions_features(ctx, m, cfg, frames_by_session, level, scale, n_slots, log_n, device, bufs=None,
                      per_call=1):
    """Partial features of this rank's frame shard for every session: one ciphertext per
    session, stacked [S, 2, level_out+1, N] (device, int64 view of the residues).  `bufs`:
    optional persistent [S, 2, level_out+1, N] output tensor (stable buffer addresses let the
    library replay its captured chain graphs from call to call).  per_call > 1: that many
    sessions' shards per gesture_features call as one batch (cfg.sessions; every session holds
    the same number of frame groups)."""
    import torch

    outs = []
    S = len(frames_by_session)
    for s0 in range(0, S, max(1, per_call)):
        chunk = frames_by_session[s0:s0 + max(1, per_call)]
        k = len(chunk)
        ccfg = cfg
        if k > 1:
            ccfg = type(cfg).from_buffer_copy(cfg)
            ccfg.sessions = k
            ins = m.CtArray([c for a in chunk for c in (a.cts if isinstance(a, m.CtArray) else a)])
        else:
            ins = chunk[0]
        lvs = ctx.chain_plan("gesture_features", ccfg, level, len(ins))
        os_ = []
        for i, lv in enumerate(lvs):
            data = bufs[s0 + i] if bufs is not None else torch.empty((2, lv + 1, 1 << log_n), dtype=torch.int64,
                                                                     device=device)
            os_.append(m.Ct(data, lv, 0.0, 0, log_n, m.FORM_EVAL))
        ctx.eval_chain("gesture_features", ccfg, ins, os_)
        outs += os_
    stacked = bufs if bufs is not None else torch.stack([o.data for o in outs])
    return stacked, outs[0].level, outs[0].scale


def reduce_partials(ctx, m, gathered, session, level, scale, n_slots, log_n, buf=None):
    """Library-side modular sum of session `session`'s partials from every rank (into the
    optional persistent tensor `buf`)."""
    import torch

    parts = [m.Ct(gathered[r, session], level, scale, n_slots, log_n, m.FORM_EVAL) for r in range(gathered.shape[0])]
    out = m.Ct(buf if buf is not None else torch.empty_like(gathered[0, session]), level, 0.0, 0, log_n,
               m.FORM_EVAL)
    ctx.sum_partials(parts, out)
    return out
