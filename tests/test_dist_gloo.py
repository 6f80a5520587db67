"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU plumbing:
sharding covers every unit exactly once, the all-gather of partial ciphertexts
returns every rank's partial in rank order, and summing the gathered partials
mod q reproduces the sum over all frames (the exchange step of P:906; the GPU
performs that sum in mmfhe_sum_partials, covered by the GPU parity tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_22437_b200.dist import allgather_partials, owner, shard

Q = (1 << 59) + 21  # any modulus < 2^61 for the stand-in sum


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames(F, shape, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, Q, size=(F,) + shape, dtype=np.int64)


def _worker(rank, world, port, F, sessions, shape, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = [_frames(F, shape, 100 + s) for s in range(sessions)]
        lo, hi = shard(F, rank, world)
        # each rank sums its own frame shard of every session (stand-in for gesture_features)
        partial = np.stack([(f[lo:hi].astype(object).sum(axis=0) % Q).astype(np.int64) for f in frames])
        gathered = allgather_partials(torch.from_numpy(partial))
        assert tuple(gathered.shape) == (world, sessions) + shape
        for s in range(sessions):
            if owner(s, world) != rank:
                continue
            total = (gathered[:, s].numpy().astype(object).sum(axis=0) % Q).astype(np.int64)
            want = (frames[s].astype(object).sum(axis=0) % Q).astype(np.int64)
            assert np.array_equal(total, want)
        # every rank's partial arrives in rank order
        for r in range(world):
            rlo, rhi = shard(F, r, world)
            want_r = np.stack([(f[rlo:rhi].astype(object).sum(axis=0) % Q).astype(np.int64) for f in frames])
            assert np.array_equal(gathered[r].numpy(), want_r)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("F,sessions", [(7, 3), (100, 2)])
def test_allgather_partial_sums_world2(F, sessions):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, F, sessions, (2, 3, 16), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (7, 2), (100, 8), (3, 8), (256, 3)])
def test_shard_covers_every_unit_once(n, world):
    seen = []
    sizes = []
    for r in range(world):
        lo, hi = shard(n, r, world)
        seen += list(range(lo, hi))
        sizes.append(hi - lo)
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def test_allgather_without_process_group_is_identity():
    x = torch.arange(12, dtype=torch.int64).reshape(3, 4)
    g = allgather_partials(x)
    assert g.shape == (1, 3, 4) and torch.equal(g[0], x)
