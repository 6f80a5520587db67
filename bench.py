#!/usr/bin/env python
"""bench.py -- encrypted frames/s of the mmFHE vital-signs pipeline on B200.

Metric (BASELINE.json): "encrypted frames/sec per pipeline; HRot & HMult
ops/sec and HBM GB/s at N=2^16".

Workload at N=1 GPU: configs[1] = C2, the vital-signs pipeline (vitals_v1 =
K1 -> K2 at entry level 3, vitals_v2 = K4 -> K5 -> K7 -> narrowband DFT ->
|X|^2 at entry level 7), N = 2^14, R = 128 range bins, F = 256 frames, PS2
(8 Q limbs + 1 P).  One step = one session: 2F ciphertexts into each chain.
Extras: HRot/s and HMult/s at N = 2^16 (PS4, 20 Q limbs, dnum 3, top level).

Inputs are seeded synthetic residues: RLWE ciphertexts and evaluation keys
are uniform mod q (IND-CPA), and the circuits are data-oblivious
(Theorem P:999-1006), so the work is that of real encryptions; correctness on
real encryptions is the job of tests/ (bit-exact vs the oracle).  Public
operands (K2 ramps, DFT coefficients, FIR taps) are encoded by the library.

Multi-GPU (torchrun): sessions are independent, so each rank runs its own
session per step; no collective on the data path (weak scaling).
"""
from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted frames/sec per pipeline; HRot & HMult ops/sec and HBM GB/s at N=2^16"
BANDS = ((0.1, 0.6), (0.8, 2.5))  # RR, HR


def band_bins(F_phase, fs, band):
    k = np.arange(F_phase // 2 + 1)
    f = k * fs / F_phase
    return [int(x) for x in k[(f >= band[0]) & (f <= band[1])]]


def c2_config():
    from synth.params import ps2
    P = ps2()
    R, F, fs = 128, 256, 20.0
    bins = [band_bins(F - 1, fs, b) for b in BANDS]
    return P, dict(R=R, F=F, fs=fs, gamma=2, p_phi=2, taylor_order=1, n_slots=P.n // 2, bins=bins, n_taps=41,
                   v1_level=3, v2_level=7, iq_pack=3, hoist=1)


def c2_bench_config(world):
    """The N=1 workload (BASELINE configs[1]) both arms report as `config`."""
    return {"workload": "C2 vital-signs pipeline: vitals_v1 (K1->K2, entry level 3) + vitals_v2 "
                        "(K4->K5->K7->narrowband DFT->|X|^2, entry level 7)",
            "N": 2 ** 14, "R": 128, "F": 256, "params": "PS2: 8 Q limbs (60+7x40) + 1 P, alpha 1",
            "sessions_per_step_per_gpu": 1, "parallelism": f"session-sharded x{world}",
            "l2": "inputs larger than L2 (1.5 GiB of ciphertexts per step)",
            "inputs": "coefficient form, device-resident; import NTT and export INTT in the step",
            "k4_rotsum": "packed I/Q rotate-and-sum over 4 frames (DESIGN reading R19, iq_pack = 3, hoist = 1: "
                         "per frame 1.75 packing + 1.75 rotate-and-sum rotations + 1.75 hoisted unpacking "
                         "rotations sharing one ModUp per 4 frames, instead of 14 rotations)"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed region,
    in-process through NVML (the same counters nvidia-smi's clocks line reads; a
    background `nvidia-smi -lms` poller measurably stalled this workload)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int, interval_s: float = 0.1):
        self.gpu = gpu_index
        self.interval = interval_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for nm, bit in self.REASONS.items():
                            if mask & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    self._stop.wait(self.interval)

            # first NVML queries cost ~0.3 s of process time: pay them before the timed region
            for _ in range(3):
                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self._thread = threading.Thread(target=run, daemon=True)
            self._thread.start()
            time.sleep(0.5)
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML, 100 ms"}


# ---------------------------------------------------------------- GPU arm
def uniform_dev(torch, gen, shape_rows, qs, n, device):
    """[..., rows, n] residues uniform mod the row's prime (rows cycle through qs)."""
    out = torch.empty(shape_rows + (n,), dtype=torch.int64, device=device)
    flat = out.view(-1, len(qs), n)
    for i, q in enumerate(qs):
        flat[:, i].random_(0, int(q), generator=gen)
    return out


def make_ctx_c2(m, torch, P, cfg, device, seed):
    ctx = m.Context.from_params(P, device=device.index or 0, stream=torch.cuda.current_stream(device).cuda_stream)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    basis = list(P.q) + list(P.p)
    key_shape = (P.dnum(), 2, len(basis))
    ctx.load_relin_key(uniform_dev(torch, gen, key_shape, basis, P.n, device))
    mcfg = chain_cfg_c2(m, cfg)
    for k in sorted(set(ctx.required_rotations("vitals_v1", mcfg) + ctx.required_rotations("vitals_v2", mcfg))):
        ctx.load_galois_key(k, uniform_dev(torch, gen, key_shape, basis, P.n, device))
    from synth.radar import fir_taps
    taps = [fir_taps(cfg["n_taps"], b, cfg["fs"]) for b in BANDS]
    ctx.prepare_chain("vitals_v2", mcfg, cfg["v2_level"], taps=taps)
    ctx.prepare_chain("vitals_v1", mcfg, cfg["v1_level"])
    return ctx, gen


def chain_cfg_c2(m, cfg):
    return m.chain_cfg(R=cfg["R"], F=cfg["F"], gamma=cfg["gamma"], p_phi=cfg["p_phi"],
                       taylor_order=cfg["taylor_order"], n_slots=cfg["n_slots"], bands_bins=cfg["bins"],
                       n_taps=[cfg["n_taps"]] * 2, fs=cfg["fs"], iq_pack=cfg.get("iq_pack", 0),
                       hoist=cfg.get("hoist", 0))


def session_inputs(m, torch, gen, P, cfg, device):
    F = cfg["F"]
    scale = float(2 ** P.scale_bits)
    ins = {}
    for chain, lvl in (("vitals_v1", cfg["v1_level"]), ("vitals_v2", cfg["v2_level"])):
        data = uniform_dev(torch, gen, (2 * F, 2, lvl + 1), list(P.q[: lvl + 1]), P.n, device)
        ins[chain] = [m.Ct(data[i], lvl, scale, cfg["n_slots"], P.log_n) for i in range(2 * F)]
    return ins


def outputs_for(m, torch, ctx, P, mcfg, chain, ins, device, host=False):
    levels = ctx.chain_plan(chain, mcfg, ins[0].level, len(ins))
    outs = []
    for lv in levels:
        if host:
            buf = np.empty((2, lv + 1, P.n), dtype=np.uint64)
        else:
            buf = torch.empty((2, lv + 1, P.n), dtype=torch.int64, device=device)
        outs.append(m.Ct(buf, lv, 0.0, 0, P.log_n))
    return outs


def run_gpu(args, rank, world, device):
    import torch
    from paper_2603_22437_b200 import mmfhe as m

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    P, cfg = c2_config()
    torch.cuda.set_device(device)
    ctx, gen = make_ctx_c2(m, torch, P, cfg, device, seed=1000 + 2 + rank)
    mcfg = chain_cfg_c2(m, cfg)
    ins = session_inputs(m, torch, gen, P, cfg, device)
    outs = {c: outputs_for(m, torch, ctx, P, mcfg, c, ins[c], device) for c in ins}
    stream = torch.cuda.current_stream(device)
    ins_a = {c: m.CtArray(ins[c]) for c in ins}      # marshalled once (binding-side cost only)
    outs_a = {c: m.CtArray(outs[c]) for c in outs}

    def step():
        for chain in ("vitals_v1", "vitals_v2"):
            ctx.eval_chain(chain, mcfg, ins_a[chain], outs_a[chain])

    ctx.trace_enable(False)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(device)
    # timed region: barrier + sync on both sides, CUDA events on the ctx stream
    if dist:
        tdist.barrier()
    torch.cuda.synchronize(device)
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index or 0) as clk:
        torch.cuda.synchronize(device)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(device)
    if dist:
        tdist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = (ctx.launch_count() - launches0) // max(args.steps, 1)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if dist:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    frames = cfg["F"] * args.steps * world
    value = frames / (ms_max / 1e3)

    # profile pass (same workload, CUDA events around every launch): roofline of the dominant kernel
    ctx.profile_enable(True)
    prof_steps = max(1, min(2, args.steps))
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(prof_steps):
        step()
    pe1.record(stream)
    prof = ctx.profile()
    ctx.profile_enable(False)
    prof_ms = pe0.elapsed_time(pe1)
    # the NTT's own butterflies (truncated-quotient Shoup, kinds 4/5) set its integer roof;
    # the exact-quotient butterflies are reported beside them
    int_peaks = {"ct_butterfly": ctx.microbench(4), "gs_butterfly": ctx.microbench(5), "mac128": ctx.microbench(2),
                 "shoup_modmul": ctx.microbench(3), "ct_butterfly_exact_quotient": ctx.microbench(0),
                 "gs_butterfly_exact_quotient": ctx.microbench(1)}

    # e2e: host buffers through the C-ABI, H2D / D2H inside the timed region
    e2e = None
    if rank == 0 or dist:
        # pinned host buffers: the session's uplink lands in one page-locked receive buffer
        # per chain (frames back to back), which the library uploads with one copy per call
        hin = {}
        for c in ins:
            stacked = torch.stack([x.data for x in ins[c]]).cpu().pin_memory()
            hin[c] = [m.Ct(stacked[i], x.level, x.scale, x.n_slots, x.log_n) for i, x in enumerate(ins[c])]
        hout = {}
        for c in ins:
            outs_h = []
            for lv in ctx.chain_plan(c, mcfg, ins[c][0].level, len(ins[c])):
                buf = torch.empty((2, lv + 1, P.n), dtype=torch.int64, pin_memory=True)
                outs_h.append(m.Ct(buf, lv, 0.0, 0, P.log_n))
            hout[c] = outs_h
        h2d = sum(x.data.numel() * 8 for c in hin for x in hin[c])
        d2h = sum(x.data.numel() * 8 for c in hout for x in hout[c])
        hin = {c: m.CtArray(hin[c]) for c in hin}
        hout = {c: m.CtArray(hout[c]) for c in hout}
        # mmfhe_eval_chain_async: the upload of step i+1 (library copy stream, two device
        # staging slots) overlaps the compute of step i; every step's H2D and D2H is
        # inside the timed region (host wall clock around the loop + final sync)
        for _ in range(4):  # both staging slots through eager run + graph capture
            for chain in hin:
                ctx.eval_chain_async(chain, mcfg, hin[chain], hout[chain])
        ctx.sync()
        e_steps = max(10, args.steps)  # the first upload cannot overlap a previous step: amortise the fill
        if dist:
            tdist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            for chain in hin:
                ctx.eval_chain_async(chain, mcfg, hin[chain], hout[chain])
        ctx.sync()
        e_s = (time.perf_counter() - t0) / e_steps
        if dist:  # the slowest rank's wall clock
            te = torch.tensor([e_s], dtype=torch.float64, device=device)
            tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
            e_s = float(te.item())
        e2e = {"value": cfg["F"] * world / e_s, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_s * 1e3, "clock": "host wall, max over ranks",
               "api": "mmfhe_eval_chain_async (pinned host buffers, copy/compute overlap across steps)"}

    extras = {}
    if not args.no_extras:
        extras = extras_n16(args, m, torch, device)
        for wl in ("C1", "C3", "C4", "C5v"):
            try:
                extras[wl] = bench_workload(wl, m, torch, device)
            except Exception as e:  # report, do not hide
                extras[wl] = {"error": f"{type(e).__name__}: {e}"}
        if dist:
            # C5's vital half: one full-depth session per rank (session sharding, no exchange);
            # aggregate over ranks with the slowest rank's device time (every rank joins the
            # reduction, a failed rank contributes +inf)
            t5 = torch.tensor([extras.get("C5v", {}).get("ms_per_step", float("inf"))], dtype=torch.float64,
                              device=device)
            tdist.all_reduce(t5, op=tdist.ReduceOp.MAX)
            if math.isfinite(float(t5.item())):
                extras["C5v"]["n_gpus"] = world
                extras["C5v"]["frames_per_s_all_ranks"] = (world * extras["C5v"]["frames_per_step"] /
                                                           (float(t5.item()) / 1e3))
    if not args.no_c5:
        extras["C5"] = bench_c5(m, torch, device, rank, world)
    return dict(value=value, ms=ms_max / args.steps, launches=launches, clocks=clk.summary(), prof=prof,
                prof_steps=prof_steps, prof_ms=prof_ms / prof_steps, e2e=e2e, extras=extras, cfg=cfg, P=P,
                int_peaks=int_peaks)


def bench_workload(name, m, torch, device, steps=2, warmup=2):
    """Encrypted frames/s of the other BASELINE.json configs (SURVEY §8(d) definitions),
    device-resident coefficient-form inputs, CUDA events on the library stream:
      C1: K1 energy, N=2^13 (PS1), R=64, F=32, 256 sessions per step (frames = sessions*F);
      C3: K3 Doppler DFT, N=2^15 (PS3), A=4 x R=32 x D=32, 32 frames per step, hoisted baby steps;
      C4: gesture session, N=2^16 (PS4, entry level 19), F=100 frames + FC 4096->64->32->5;
      C5v: one vital session of C5 at full depth, N=2^16 (PS4), R=64, F=200 @ 20 Hz: vitals_v1
           (entry level 3) + vitals_v2 first order with VP+ in the cloud (entry level 9, depth 9)."""
    from synth import radar
    from synth.params import ps1, ps3, ps4
    stream = torch.cuda.current_stream(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(7000 + ord(name[1]))
    if name == "C1":
        P = ps1()
        cfg = m.chain_cfg(R=64, F=32, n_slots=P.n // 2)
        chain, lvl, n_in, frames, info = "k1_energy", 1, 2 * 32 * 256, 32 * 256, "256 sessions x F=32"
    elif name == "C3":
        P = ps3()
        cfg = m.chain_cfg(A=4, R=32, D=32, n_slots=4096, frame_batch=32, hoist=1)
        chain, lvl, n_in, frames, info = "k3_doppler_dft", P.L, 64, 32, "32 frames, frame_batch 32, hoisted"
    elif name == "C4":
        P = ps4()
        cfg = m.chain_cfg(A=4, R=32, D=32, F=100, gamma=4, n_slots=4096, fc_dims=(4096, 64, 32, 8),
                          frame_batch=25, hoist=1)
        chain, lvl, n_in, frames, info = "gesture", 19, 200, 100, "F=100 frames, frame_batch 25, hoisted"
    else:
        P = ps4()
        F, fs = 200, 20.0
        cfg = m.chain_cfg(R=64, F=F, gamma=2, p_phi=2, taylor_order=1, n_slots=P.n // 2,
                          bands_bins=[band_bins(F - 1, fs, b) for b in BANDS], n_taps=[41, 41], fs=fs,
                          frame_batch=40, vp_plus=1, iq_pack=3, hoist=1)
        chain, lvl, n_in, frames, info = "vitals_v2", 9, 2 * F, F, "F=200 frames, frame_batch 40, VP+ in the cloud"
    # one step = these chain calls (C5v: V1 then V2 on the same session's frames)
    plan = [("vitals_v1", 3, n_in), (chain, lvl, n_in)] if name == "C5v" else [(chain, lvl, n_in)]
    ctx = m.Context.from_params(P, device=device.index or 0, stream=stream.cuda_stream)
    basis = list(P.q) + list(P.p)
    key_shape = (P.dnum(), 2, len(basis))
    ctx.load_relin_key(uniform_dev(torch, gen, key_shape, basis, P.n, device))
    for k in sorted({k for ch, _, _ in plan for k in ctx.required_rotations(ch, cfg)}):
        ctx.load_galois_key(k, uniform_dev(torch, gen, key_shape, basis, P.n, device))
    fc_w = fc_b = None
    if chain == "gesture":
        Ws, bs = radar.fc_weights([4096, 64, 32, 5], seed=11)
        Ws[-1] = np.vstack([Ws[-1], np.zeros((3, 32))])
        bs[-1] = np.concatenate([bs[-1], np.zeros(3)])
        fc_w, fc_b = Ws, bs
    taps = [radar.fir_taps(41, b, 20.0) for b in BANDS] if chain == "vitals_v2" else None
    scale = float(2 ** P.scale_bits)
    runs = []
    for ch, lv0, n in plan:
        ctx.prepare_chain(ch, cfg, lv0, fc_w=fc_w, fc_b=fc_b, taps=taps if ch == "vitals_v2" else None)
        data = uniform_dev(torch, gen, (n, 2, lv0 + 1), list(P.q[: lv0 + 1]), P.n, device)
        ins = m.CtArray([m.Ct(data[i], lv0, scale, cfg.n_slots, P.log_n) for i in range(n)])
        outs = m.CtArray([m.Ct(torch.empty((2, lv + 1, P.n), dtype=torch.int64, device=device), lv, 0.0, 0,
                               P.log_n) for lv in ctx.chain_plan(ch, cfg, lv0, n)])
        runs.append((ch, ins, outs, data))

    def step():
        for ch, ins, outs, _ in runs:
            ctx.eval_chain(ch, cfg, ins, outs)

    ctx.trace_enable(False)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(device)
    l0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(device)
    ms = e0.elapsed_time(e1) / steps
    launches = (ctx.launch_count() - l0) // steps
    ctx.profile_enable(True)
    step()
    prof = ctx.profile()
    ctx.profile_enable(False)
    top = sorted(prof.items(), key=lambda kv: -kv[1][1])[:6]
    res = {"frames_per_s": frames / (ms / 1e3), "ms_per_step": ms, "frames_per_step": frames,
           "gpu_launches_per_step": launches,
           "kernel_ms_top": {k: round(v[1], 3) for k, v in top},
           "kernel_ms_total": round(sum(v[1] for v in prof.values()), 3),
           "config": f"{' + '.join(ch for ch, _, _ in plan)} at N=2^{P.log_n} ({len(P.q)} Q + {len(P.p)} P limbs, "
                     f"entry level {' / '.join(str(lv) for _, lv, _ in plan)}), {info}"}
    ctx.close()
    del runs
    torch.cuda.empty_cache()
    return res


def bench_c5(m, torch, device, rank, world, sessions_per_rank=1, F=100, steps=2, warmup=2):
    """C5 batched multi-session gesture serving (BASELINE configs[4]) with the method's one
    exchange step: G = sessions_per_rank * world sessions per step; every session's F
    frames are sharded over the ranks (paper_2603_22437_b200.dist.shard); each rank runs
    gesture_features on its shard of every session, the per-rank partial feature
    ciphertexts are all-gathered over NCCL, and the owner of each session sums them in the
    library (mmfhe_sum_partials) and runs the FC head.  Weak scaling: per-rank work is
    fixed (F frames + sessions_per_rank FC heads per step)."""
    from paper_2603_22437_b200 import dist as mdist
    from synth import radar
    from synth.params import ps4
    import torch.distributed as tdist
    distributed = tdist.is_available() and tdist.is_initialized()
    P = ps4()
    lvl = 19
    stream = torch.cuda.current_stream(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(9100)  # same keys on every rank (the client's key set, replicated)
    cfg = m.chain_cfg(A=4, R=32, D=32, F=F, gamma=4, n_slots=4096, fc_dims=(4096, 64, 32, 8), frame_batch=25,
                      hoist=1)
    ctx = m.Context.from_params(P, device=device.index or 0, stream=stream.cuda_stream)
    basis = list(P.q) + list(P.p)
    key_shape = (P.dnum(), 2, len(basis))
    ctx.load_relin_key(uniform_dev(torch, gen, key_shape, basis, P.n, device))
    for k in ctx.required_rotations("gesture", cfg):
        ctx.load_galois_key(k, uniform_dev(torch, gen, key_shape, basis, P.n, device))
    Ws, bs = radar.fc_weights([4096, 64, 32, 5], seed=11)
    Ws[-1] = np.vstack([Ws[-1], np.zeros((3, 32))])
    bs[-1] = np.concatenate([bs[-1], np.zeros(3)])
    ctx.prepare_chain("gesture", cfg, lvl, fc_w=Ws, fc_b=bs)
    G = sessions_per_rank * world
    lo, hi = mdist.shard(F, rank, world)
    gen_in = torch.Generator(device=device)
    gen_in.manual_seed(9200 + rank)
    scale = float(2 ** P.scale_bits)
    data = uniform_dev(torch, gen_in, (G, 2 * (hi - lo), 2, lvl + 1), list(P.q[: lvl + 1]), P.n, device)
    frames_by_session = [m.CtArray([m.Ct(data[s, i], lvl, scale, 4096, P.log_n) for i in range(2 * (hi - lo))])
                         for s in range(G)]
    mine = [s for s in range(G) if mdist.owner(s, world) == rank]
    ctx.trace_enable(False)
    # persistent chain output buffers: stable addresses, so the library's chain graphs are
    # captured during warm-up and replayed in the timed steps (never captured inside them)
    lvf = ctx.chain_plan("gesture_features", cfg, lvl, len(frames_by_session[0]))[0]
    lvo = ctx.chain_plan("gesture_fc", cfg, lvf, 1)[0]
    feat_bufs = torch.empty((G, 2, lvf + 1, P.n), dtype=torch.int64, device=device)
    sum_bufs = {s: torch.empty((2, lvf + 1, P.n), dtype=torch.int64, device=device) for s in mine}
    fc_outs = {s: m.Ct(torch.empty((2, lvo + 1, P.n), dtype=torch.int64, device=device), lvo, 0.0, 0, P.log_n,
                       m.FORM_EVAL) for s in mine}

    def step():
        partials, lv, sc = mdist.sessions_features(ctx, m, cfg, frames_by_session, lvl, scale, 4096, P.log_n, device,
                                                   bufs=feat_bufs)
        gathered = mdist.allgather_partials(partials)
        for s in mine:
            total = mdist.reduce_partials(ctx, m, gathered, s, lv, sc, 4096, P.log_n, buf=sum_bufs[s])
            ctx.eval_chain("gesture_fc", cfg, [total], [fc_outs[s]])
        return partials.numel() * 8

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(device)
    if distributed:
        tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        xbytes = step()
    e1.record(stream)
    torch.cuda.synchronize(device)
    if distributed:
        tdist.barrier()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if distributed:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    ctx.close()
    del data, frames_by_session
    torch.cuda.empty_cache()
    return {"frames_per_s": G * F / (ms / 1e3), "ms_per_step": ms, "sessions_per_step": G, "frames_per_session": F,
            "n_gpus": world, "allgather_bytes_per_rank_per_step": xbytes,
            "config": "PS4 gesture sessions, frames sharded over ranks, NCCL all-gather of partial feature "
                      "ciphertexts + library mod-q sum + FC on the owning rank; weak scaling in sessions"}


def extras_n16(args, m, torch, device, batch=8, reps=3):
    """HRot/s and HMult/s at N = 2^16 (PS4, top level, independent ciphertexts, one key)."""
    from synth.params import ps4
    P = ps4()
    ctx = m.Context.from_params(P, device=device.index or 0, stream=torch.cuda.current_stream(device).cuda_stream)
    gen = torch.Generator(device=device)
    gen.manual_seed(4242)
    basis = list(P.q) + list(P.p)
    key_shape = (P.dnum(), 2, len(basis))
    ctx.load_relin_key(uniform_dev(torch, gen, key_shape, basis, P.n, device))
    ctx.load_galois_key(1, uniform_dev(torch, gen, key_shape, basis, P.n, device))
    L = P.L
    scale = float(2 ** P.scale_bits)
    # inputs in the library's evaluation form, device-resident (no import/export in the op timing)
    data = uniform_dev(torch, gen, (batch, 2, L + 1), list(P.q), P.n, device)
    cts = [m.Ct(data[i], L, scale, P.n // 2, P.log_n, m.FORM_EVAL) for i in range(batch)]
    data2 = uniform_dev(torch, gen, (batch, 2, L + 1), list(P.q), P.n, device)
    cts2 = [m.Ct(data2[i], L, scale, P.n // 2, P.log_n, m.FORM_EVAL) for i in range(batch)]
    obuf = torch.empty((batch, 2, L + 1, P.n), dtype=torch.int64, device=device)
    outs = [m.Ct(obuf[i], L, 0.0, 0, P.log_n, m.FORM_EVAL) for i in range(batch)]
    ctx.trace_enable(False)
    stream = torch.cuda.current_stream(device)
    res = {}
    limb = P.n * 8
    evk = P.dnum() * 2 * (L + 1 + P.K) * limb
    ct_bytes = 2 * (L + 1) * limb
    for name, fn, alg in (("hrot", lambda: ctx.hrot_batch(cts, 1, outs), 2 * ct_bytes + evk),
                          ("hmult", lambda: ctx.hmult_batch(cts, cts2, outs), 3 * ct_bytes + evk)):
        fn()
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(device)
        s = e0.elapsed_time(e1) / 1e3
        ops = batch * reps / s
        res[f"{name}_per_s"] = ops
        res[f"{name}_us"] = 1e6 / ops
        res[f"{name}_alg_gbs"] = ops * alg / 1e9
    # SURVEY §8(d) variants 2 and 3: one ciphertext per op (the 81 MiB evk streamed for every
    # rotation: the worst case) and a hoisted group of 8 rotations of one ciphertext
    # batch 64 sharing the key (SURVEY §8(d) metric 2: "batch 1 and batch 64 sharing a key")
    data64 = uniform_dev(torch, gen, (64, 2, L + 1), list(P.q), P.n, device)
    cts64 = [m.Ct(data64[i], L, scale, P.n // 2, P.log_n, m.FORM_EVAL) for i in range(64)]
    obuf64 = torch.empty((64, 2, L + 1, P.n), dtype=torch.int64, device=device)
    outs64 = [m.Ct(obuf64[i], L, 0.0, 0, P.log_n, m.FORM_EVAL) for i in range(64)]
    ctx.hrot_batch(cts64, 1, outs64)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.hrot_batch(cts64, 1, outs64)
    e1.record(stream)
    torch.cuda.synchronize(device)
    s64 = e0.elapsed_time(e1) / 1e3
    res["hrot_b64_us"] = s64 / 64 * 1e6
    res["hrot_b64_alg_gbs"] = (64 * 2 * ct_bytes + evk) / s64 / 1e9
    del data64, obuf64, cts64, outs64
    steps8 = list(range(1, 9))
    for k in steps8[1:]:
        ctx.load_galois_key(k, uniform_dev(torch, gen, key_shape, basis, P.n, device))
    one, oone = cts[0], outs[0]
    houts = [m.Ct(obuf[i], L, 0.0, 0, P.log_n, m.FORM_EVAL) for i in range(8)]
    for name, fn, n_ops, alg in (("hrot_b1", lambda: ctx.hrot_batch([one], 1, [oone]), 1, 2 * ct_bytes + evk),
                                 ("hrot_hoisted8", lambda: ctx.hrot_hoisted(one, steps8, houts), 8,
                                  ct_bytes + 8 * (evk + ct_bytes))):
        fn()
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(device)
        s = e0.elapsed_time(e1) / 1e3 / reps
        res[f"{name}_us_per_rotation"] = s / n_ops * 1e6
        res[f"{name}_alg_gbs"] = alg / s / 1e9
    # integer roof: the key switch's algorithmic butterflies, 128-bit MACs and
    # modular products against the butterfly / MAC / Shoup rates measured in this run
    Lp, K, N, logn = L + 1, P.K, P.n, P.log_n
    bn = N // 2 * logn
    alphas = [min(P.alpha, Lp - j * P.alpha) for j in range(P.dnum())]
    bfly = Lp * bn + sum(Lp + K - a for a in alphas) * bn + 2 * K * bn + 2 * Lp * bn
    mac = sum(a * (Lp + K - a + 1) for a in alphas) * N + len(alphas) * 2 * (Lp + K) * N + 2 * K * (Lp + 1) * N
    mm = 2 * Lp * N
    peaks = {"bfly": ctx.microbench(4), "mac": ctx.microbench(2), "mm": ctx.microbench(3)}
    t_int = bfly / peaks["bfly"] + mac / peaks["mac"] + mm / peaks["mm"]
    for name, extra_mac in (("hrot", 0), ("hmult", 4 * Lp * N)):
        t = t_int + extra_mac / peaks["mac"]
        res[f"{name}_int_model_us"] = t * 1e6
        res[f"{name}_int_frac"] = t * res[f"{name}_per_s"]
    res["int_model"] = (f"per key switch: {bfly / 1e6:.1f} M butterflies + {mac / 1e6:.1f} M MAC128 + {mm / 1e6:.1f} M "
                        f"modmul (SURVEY 8(d)); HMult adds 4L'N tensor MACs; peaks measured in this run: "
                        f"{peaks['bfly'] / 1e9:.0f} G bfly/s, {peaks['mac'] / 1e9:.0f} G MAC/s, "
                        f"{peaks['mm'] / 1e9:.0f} G modmul/s; int_frac = model time / measured time")
    res["config"] = ("PS4: N=2^16, 20 Q + 7 P limbs, dnum 3, top level, eval form; hrot/hmult: batch of 8 "
                     "distinct cts, one key; hrot_b64: batch of 64 sharing the key; hrot_b1: one ct per call; hrot_hoisted8: steps 1..8 of one ct "
                     "(one ModUp, 8 inner products + ModDowns, 8 keys)")
    ctx.close()
    return res


# ---------------------------------------------------------------- oracle (CPU) arms
def oracle_sample(frames: int, threads: int):
    """Time the oracle (as it stands) on a bounded sample of the C2 workload:
    vitals_v1 and vitals_v2 on `frames` frames (uniform residues / keys, as the
    GPU arm), K4 frames spread over `threads` host threads.  Returns (seconds, frames)."""
    import concurrent.futures as cf

    from oracle import ckks as orc
    from oracle import circuits as cc
    from synth import prng

    P, cfg = c2_config()
    rng_seed = 77
    basis = list(P.q) + list(P.p)

    def ukey(sid):
        out = np.empty((P.dnum(), 2, len(basis), P.n), dtype=np.uint64)
        for j in range(P.dnum()):
            for p in range(2):
                for t, q in enumerate(basis):
                    out[j, p, t] = prng.uniform_mod(rng_seed, sid + 4 * j + p, P.n, q, offset=t * P.n)
        return out

    ccfg = cc.ChainCfg(R=cfg["R"], F=frames, gamma=2, p_phi=2, taylor_order=1, n_slots=cfg["n_slots"],
                       fs=cfg["fs"], bands=BANDS, iq_pack=cfg.get("iq_pack", 0), hoist=cfg.get("hoist", 0))
    rots = cc.required_rotations("vitals_v2", ccfg, P.n)
    rlk = ukey(prng.SID_UNIFORM)
    gk = {k: ukey(prng.SID_UNIFORM + 100 * (i + 1)) for i, k in enumerate(rots)}

    def uct(level, idx):
        c = [np.stack([prng.uniform_mod(rng_seed, prng.SID_UNIFORM + 10 ** 6 + 4 * idx + p, P.n, q, offset=i * P.n)
                       for i, q in enumerate(P.q[: level + 1])]) for p in range(2)]
        return orc.Ct(c, level, float(2 ** P.scale_bits), cfg["n_slots"])

    v1 = [uct(cfg["v1_level"], i) for i in range(2 * frames)]
    v2 = [uct(cfg["v2_level"], 1000 + i) for i in range(2 * frames)]
    from synth.radar import fir_taps
    taps = [fir_taps(cfg["n_taps"], b, cfg["fs"]) for b in BANDS]
    t0 = time.perf_counter()
    ev = cc.CircuitEvaluator(P, rlk, gk)
    cc.vitals_v1(ev, cc.PlainBook(P), v1[0::2], v1[1::2], ccfg)

    # K4 in groups of 2^(iq_pack - 1) frames (the packed rotate-and-sum's unit), groups on threads
    g = 1 << max(ccfg.iq_pack - 1, 0)

    def k4(t0):
        e = cc.CircuitEvaluator(P, rlk, gk)
        return cc.k4_soft_iq(e, v2[2 * t0:2 * (t0 + g):2], v2[2 * t0 + 1:2 * (t0 + g):2], ccfg)

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        IQ = list(ex.map(k4, range(0, frames, g)))
    I, Q = [x for a, _ in IQ for x in a], [x for _, b in IQ for x in b]
    for bi, h in enumerate(taps):
        If, Qf = cc.k5_fir(ev, I, h), cc.k5_fir(ev, Q, h)
        ys = cc.k7_taylor_phase(ev, If, Qf, 1)
        bins = band_bins(len(ys), cfg["fs"], BANDS[bi]) or [1]  # short samples: keep >= 1 bin
        cc.vp_band_power(ev, ys, bins)
    return time.perf_counter() - t0, frames


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores."""
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    frames = args.ref_frames
    for _ in range(args.warmup):
        oracle_sample(frames, threads)
    secs = 0.0
    n = 0
    for _ in range(args.steps):
        s, f = oracle_sample(frames, threads)
        secs += s
        n += f
    v = n / secs
    sample = (f"vitals_v1 + vitals_v2 on {frames} of the C2 session's F=256 frames per step "
              f"(PS2, N=2^14, R=128, same chain config), K4 in groups of 4 frames on "
              f"{min(threads, max(frames // 4, 1))} threads; "
              f"frames/s = frames / seconds")
    return {"metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "impl": "reference",
            "config": c2_bench_config(world),
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": min(threads, max(frames // 4, 1)), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------- main
def roofline(prof, peaks, int_peaks):
    """Dominant kernel (largest total time in the profiled steps).  NTT passes are
    integer-ALU bound: achieved butterflies/s against the butterfly
    rate measured in this run by the register-resident microbenchmark
    (mmfhe_microbench); every other kernel against the measured HBM peak."""
    if not prof:
        return None
    # group by CUDA kernel: the ModDown / rescale epilogue launches ("ntt_fwd_row_epi") are
    # the forward row-pass kernel in its epilogue mode (ncu's launch list counts them together)
    groups = {}
    for nm, (c_, m_, b_, o_) in prof.items():
        key = "ntt_fwd_row" if nm.startswith("ntt_fwd_row") else nm
        g = groups.setdefault(key, [0, 0.0, 0.0, 0.0])
        g[0] += c_
        g[1] += m_
        g[2] += b_
        g[3] += o_
    name, (cnt, ms, by, ops) = max(groups.items(), key=lambda kv: kv[1][1])
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    share = ms / sum(v[1] for v in prof.values())
    gbs = by / (ms / 1e3) / 1e9
    out = {"kernel": name + (" (incl. its ModDown/rescale epilogue launches)" if name == "ntt_fwd_row" and
                              "ntt_fwd_row_epi" in prof else ""),
           "launches_profiled": cnt, "avg_launch_us": ms * 1e3 / max(cnt, 1),
           "share_of_kernel_time": share, "alg_bytes_per_launch": by / max(cnt, 1),
           "hbm_achieved_gbs": gbs, "hbm_frac": gbs / hbm_peak, "traffic": None}
    if name.startswith("ntt_") and ops > 0:
        peak = int_peaks["ct_butterfly"] if "fwd" in name else int_peaks["gs_butterfly"]
        ach = ops / (ms / 1e3)
        out.update({"bound": "alu", "achieved": ach / 1e9, "peak": peak / 1e9, "unit": "Gbutterfly/s",
                    "frac": ach / peak, "alg_ops_per_launch": ops / max(cnt, 1),
                    "peak_source": "measured in this run: mmfhe_microbench register-resident "
                                   + ("CT" if "fwd" in name else "GS")
                                   + " butterflies (the NTT's truncated-quotient Shoup product) over the whole GPU"})
    else:
        out.update({"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                    "peak_source": hbm_src})
    # DRAM traffic from the committed ncu --set full capture of this kernel (dram read +
    # write per launch / algorithmic bytes of that launch), applied to this run's launches
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "ncu_traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath)).get("kernels", {}).get(name)
        if tr:
            out["traffic"] = tr["ratio"] * by / max(cnt, 1)
            out["traffic_source"] = (f"{tr['capture']}: {tr['dram_bytes']} B DRAM for {tr['alg_bytes']} B algorithmic "
                                     f"({tr['launch']}); ratio {tr['ratio']} x this run's bytes per launch")
    return out


def kernel_table(prof, peaks, int_peaks, steps):
    """Per kernel: ms/step, algorithmic HBM GB/s and its fraction of the measured HBM peak;
    NTT passes also Gbutterfly/s against the in-run butterfly microbenchmark."""
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    out = {}
    for name, (cnt, ms, by, ops) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        gbs = by / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        row = {"ms_per_step": round(ms / steps, 3), "launches_per_step": cnt // max(steps, 1),
               "alg_gbs": round(gbs, 1), "hbm_frac": round(gbs / hbm_peak, 3)}
        if name.startswith("ntt_") and ops > 0 and ms > 0:
            peak = int_peaks["ct_butterfly"] if "fwd" in name else int_peaks["gs_butterfly"]
            row["gbfly_s"] = round(ops / (ms / 1e3) / 1e9, 1)
            row["alu_frac"] = round(ops / (ms / 1e3) / peak, 3)
        out[name] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mmfhe", "reference"], default="mmfhe")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the multi-GPU C5 exchange workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-frames", type=int, default=16)
    ap.add_argument("--profile-out", default="")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "mmfhe" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch
    # one process per GPU; MMFHE_BENCH_BACKEND=gloo (ranks sharing a GPU) only checks the
    # multi-rank logic on a one-GPU box -- its timings are not a scaling measurement
    backend = os.environ.get("MMFHE_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend == "gloo" else local
    if world > 1:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group(backend)
    device = torch.device("cuda", local)
    r = run_gpu(args, rank, world, device)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    if rank == 0:
        P, cfg = r["P"], r["cfg"]
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            secs, frames = oracle_sample(16, threads)
            cpu = {"value": frames / secs, "unit": "frames/s", "cores": min(threads, frames // 4), "kind": "oracle",
                   "sample": f"vitals_v1 + vitals_v2 on {frames} of 256 frames (C2, PS2, same chain config), "
                             f"K4 in groups of 4 frames (the packed rotate-and-sum unit) on {min(threads, frames // 4)} "
                             f"threads, "
                             f"{secs:.1f} s wall"}
        rl = roofline(r["prof"], peaks, r["int_peaks"])
        out = {
            "metric": METRIC, "value": r["value"], "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": c2_bench_config(world),
            "clocks": r["clocks"], "e2e": r["e2e"], "gpu_launches": r["launches"], "roofline": rl,
            "cpu_baseline": cpu, "extras": r["extras"],
            "kernel_profile_ms_per_step": {k: round(v[1] / r["prof_steps"], 3) for k, v in r["prof"].items()},
            "kernel_roofline": kernel_table(r["prof"], peaks, r["int_peaks"], r["prof_steps"]),
            "profiled_step_ms": r["prof_ms"],
            "int_peaks_ops_per_s": r["int_peaks"],
        }
        if args.profile_out:
            with open(args.profile_out, "w") as f:
                json.dump(r["prof"], f, indent=1)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as tdist
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
