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


# ------------------------------------------------------------------ the exchange with real CKKS partials

class OracleCtx:
    """CPU stand-in for the library context behind paper_2603_22437_b200.dist (no GPU here):
    chain_plan / eval_chain("gesture_features") / sum_partials computed by the oracle, so the
    dist functions move and sum real partial ciphertexts."""

    def __init__(self, P, keys, book, cfg):
        from oracle import circuits as cc
        self.cc, self.P, self.keys, self.book, self.cfg = cc, P, keys, book, cfg

    def chain_plan(self, chain, cfg, level, n_in):
        assert chain == "gesture_features" and n_in % 2 == 0
        return [level - 6]

    def _ct(self, x):
        from oracle import ckks as orc
        d = x.data.numpy().view(np.uint64)
        return orc.Ct([d[0].copy(), d[1].copy()], x.level, x.scale, x.n_slots)

    def eval_chain(self, chain, cfg, ins, outs):
        cc = self.cc
        cts = [self._ct(x) for x in ins]
        ev = cc.CircuitEvaluator(self.P, self.keys.rlk, self.keys.gk)
        f = cc.gesture_features(ev, self.book, cts[0::2], cts[1::2], self.cfg)
        outs[0].data.copy_(torch.from_numpy(np.stack(f.c).view(np.int64)))
        outs[0].level, outs[0].scale = f.level, f.scale

    def sum_partials(self, parts, out):
        cc = self.cc
        ev = cc.CircuitEvaluator(self.P)
        cts = [self._ct(p) for p in parts]
        s = cc.frame_accumulate(ev, cts)
        out.data.copy_(torch.from_numpy(np.stack(s.c).view(np.int64)))
        out.level, out.scale = s.level, s.scale


def _gesture_world(seed):
    from oracle import ckks as orc
    from oracle import circuits as cc
    from synth import radar
    from synth.params import toy
    P = toy(log_n=10, n_q=8, scale_bits=40, n_p=2, alpha=2)
    n, L, F = 64, 2, 5
    cfg = cc.ChainCfg(A=2, R=4, D=8, F=F, gamma=4, n_slots=n, fc_dims=(n, 16, 8, 8), hoist=1, lanes=L)
    keys = orc.keygen(P, seed=seed, rotations=cc.required_rotations("gesture", cfg, P.n))
    sessions = []
    for s in range(3):
        Z, _ = radar.gesture_scene(2, 4, 8, F, seed=seed + 10 * s, cls=s)
        vs = [radar.pack_doppler(z) for z in radar.preprocess_gesture(Z)]
        cts = []
        for g in range(cc.n_packed(F, L)):
            for part in ("real", "imag"):
                vec = cc.interleave([getattr(v, part) for v in vs[g * L:(g + 1) * L]], L, n)
                cts.append(orc.encrypt_vector(P, keys, vec, P.L, seed=seed + 1, index=100 * s + len(cts)))
        sessions.append(cts)
    return P, cfg, keys, sessions


def _exchange_worker(rank, world, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import circuits as cc
        from paper_2603_22437_b200 import dist as mdist
        from paper_2603_22437_b200 import mmfhe as m
        P, cfg, keys, sessions = _gesture_world(seed)
        book = cc.PlainBook(P)
        ctx = OracleCtx(P, keys, book, cfg)
        npairs = len(sessions[0]) // 2
        lo, hi = mdist.shard(npairs, rank, world)

        def as_ct(c):
            return m.Ct(torch.from_numpy(np.stack(c.c).view(np.int64)), c.level, c.scale, c.n_slots, P.log_n)

        mine = [[as_ct(c) for c in s[2 * lo:2 * hi]] for s in sessions]
        bufs = torch.empty((len(sessions), 2, P.L - 6 + 1, P.n), dtype=torch.int64)
        partials, lv, sc = mdist.sessions_features(ctx, m, cfg, mine, P.L, sessions[0][0].scale, cfg.n_slots * 2,
                                                   P.log_n, "cpu", bufs=bufs)
        gathered = mdist.allgather_partials(partials)
        assert tuple(gathered.shape[:2]) == (world, len(sessions))
        for s in range(len(sessions)):
            if mdist.owner(s, world) != rank:
                continue
            total = mdist.reduce_partials(ctx, m, gathered, s, lv, sc, cfg.n_slots * 2, P.log_n)
            # the single-process oracle over all of the session's frames: equal residues
            ev = cc.CircuitEvaluator(P, keys.rlk, keys.gk)
            want = cc.gesture_features(ev, cc.PlainBook(P), sessions[s][0::2], sessions[s][1::2], cfg)
            assert total.level == want.level and total.scale == want.scale
            assert np.array_equal(total.data.numpy().view(np.uint64), np.stack(want.c))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_frame_sharded_exchange_with_ckks_partials_world2():
    """SURVEY §8(e) through paper_2603_22437_b200.dist itself (shard, sessions_features,
    allgather_partials over gloo, owner, reduce_partials) with real partial feature
    ciphertexts (oracle-backed context): every owner's reduced features equal the
    single-process gesture_features residue for residue (exact modular sums)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, 4401, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[1] for r in res) == ["ok", "ok"], res
