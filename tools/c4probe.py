"""C4 gesture step at N = 2^16 (PS4, entry level 19) on uniform-residue inputs, for ncu
captures and per-kernel CUDA-event profiles.  Usage:
    python tools/c4probe.py [--frames 25] [--steps 1] [--profile]"""
import argparse
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
from synth import radar  # noqa: E402
from synth.params import PARAM_SETS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=25)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--lanes", type=int, default=1)
ap.add_argument("--hoist", type=int, default=1)
ap.add_argument("--params", default="PS4")
ap.add_argument("--bsgs", type=int, default=0, help="K3 baby steps b (0: ceil(sqrt(2D-1)))")
ap.add_argument("--fc-baby", type=int, default=0)
ap.add_argument("--cplx", type=int, default=0, help="complex slots (DESIGN R28)")
ap.add_argument("--aligned", type=int, default=0, help="K3 giants at multiples of b (DESIGN R29)")
ap.add_argument("--inner", type=int, default=0, help="double-hoisted rotate-and-sum first level (R27; 0 = 8)")
ap.add_argument("--hoist-all", type=int, default=0, help="every rotate-and-sum level hoisted (R30)")
ap.add_argument("--merge", type=int, default=0, help="relin / ModDown + rescale as one division (R31)")
ap.add_argument("--fuse", type=int, default=0, help="K1 as one conjugate-product key switch (R32)")
ap.add_argument("--chains", default="", help="comma-separated extra chains to profile on the session's inputs "
                                             "(k3_doppler_dft, gesture_frame)")
ap.add_argument("--fc-sessions", default="", help="comma-separated session counts: profile gesture_fc over "
                "that many sessions' features as one batch")
ap.add_argument("--split", action="store_true", help="also profile gesture_features and gesture_fc on their own")
args = ap.parse_args()

dev = torch.device("cuda", 0)
P = PARAM_SETS[args.params]()
F = args.frames
stream = torch.cuda.current_stream(dev)
cfg = m.chain_cfg(A=4, R=32, D=32, F=F, gamma=4, n_slots=4096, fc_dims=(4096, 64, 32, 8),
                  frame_batch=25 if args.lanes == 1 else 0, hoist=args.hoist, lanes=args.lanes, bsgs_baby=args.bsgs,
                  fc_baby=args.fc_baby, cplx=args.cplx, bsgs_aligned=args.aligned,
                  rotsum_inner=args.inner, rotsum_hoist_all=args.hoist_all,
                  ks_merge=args.merge, k1_conj_fuse=args.fuse)
ctx = m.Context.from_params(P, device=0, stream=stream.cuda_stream)
gen = torch.Generator(device=dev)
gen.manual_seed(77)
basis = list(P.q) + list(P.p)
key_shape = (P.dnum(), 2, len(basis))
ctx.load_relin_key(bench.uniform_dev(torch, gen, key_shape, basis, P.n, dev))
for k in ctx.required_rotations("gesture", cfg):
    ctx.load_galois_key(k, bench.uniform_dev(torch, gen, key_shape, basis, P.n, dev))
Ws, bs = radar.fc_weights([4096, 64, 32, 5], seed=11)
Ws[-1] = np.vstack([Ws[-1], np.zeros((3, 32))])
bs[-1] = np.concatenate([bs[-1], np.zeros(3)])
ctx.prepare_chain("gesture", cfg, 19, fc_w=Ws, fc_b=bs)
n_in = (1 if args.cplx else 2) * -(-F // max(args.lanes, 1))
data = bench.uniform_dev(torch, gen, (n_in, 2, 20), list(P.q[:20]), P.n, dev)
ins = m.CtArray([m.Ct(data[i], 19, 2.0 ** P.scale_bits, cfg.n_slots * max(args.lanes, 1), P.log_n)
                  for i in range(n_in)])
outs = m.CtArray([m.Ct(torch.empty((2, lv + 1, P.n), dtype=torch.int64, device=dev), lv, 0.0, 0, P.log_n)
                  for lv in ctx.chain_plan("gesture", cfg, 19, n_in)])
ctx.trace_enable(False)
ctx.graph_enable(False)
for _ in range(args.steps):
    ctx.eval_chain("gesture", cfg, ins, outs)
torch.cuda.synchronize()
if args.profile:
    ctx.profile_enable(True)
    ctx.profile()
    ctx.eval_chain("gesture", cfg, ins, outs)
    prof = ctx.profile()
    tot = sum(v[1] for v in prof.values())
    print(f"gesture F={F}: kernel sum {tot:.2f} ms ({tot / F:.3f} ms/frame)")
    for k, (c, ms, by, ops) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:16s} {ms:8.2f} ms {ms / tot:6.3f}  {c:5d} launches  {by / (ms * 1e-3) / 1e9:7.1f} GB/s")

if args.profile and args.split:
    # the per-frame part (K3 -> K1 -> K6 -> K2b, pair sum) and the FC head (lane sum + 3 layers)
    fo = m.CtArray([m.Ct(torch.empty((2, lv + 1, P.n), dtype=torch.int64, device=dev), lv, 0.0, 0, P.log_n)
                    for lv in ctx.chain_plan("gesture_features", cfg, 19, n_in)])
    stages = [("gesture_features", ins, fo)]
    lf = ctx.chain_plan("gesture_features", cfg, 19, n_in)[0]
    fc_out = m.CtArray([m.Ct(torch.empty((2, lv + 1, P.n), dtype=torch.int64, device=dev), lv, 0.0, 0, P.log_n)
                        for lv in ctx.chain_plan("gesture_fc", cfg, lf, 1)])
    stages.append(("gesture_fc", fo, fc_out))
    for name, i_, o_ in stages:
        ctx.eval_chain(name, cfg, i_, o_)
        torch.cuda.synchronize()
        ctx.profile()
        ctx.eval_chain(name, cfg, i_, o_)
        prof = ctx.profile()
        tot = sum(v[1] for v in prof.values())
        print(f"{name}: kernel sum {tot:.2f} ms")
        for k, (c, ms, by, ops) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
            print(f"   {k:16s} {ms:8.2f} ms {ms / tot:6.3f}  {c:5d} launches  {by / (ms * 1e-3) / 1e9:7.1f} GB/s")

for name in [c for c in args.chains.split(",") if c]:
    lv = ctx.chain_plan(name, cfg, 19, n_in)
    o_ = m.CtArray([m.Ct(torch.empty((2, l + 1, P.n), dtype=torch.int64, device=dev), l, 0.0, 0, P.log_n) for l in lv])
    ctx.eval_chain(name, cfg, ins, o_)
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    ctx.profile()
    ctx.eval_chain(name, cfg, ins, o_)
    prof = ctx.profile()
    tot = sum(v[1] for v in prof.values())
    print(f"{name}: kernel sum {tot:.2f} ms")
    for k, (c, ms, by, ops) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:16s} {ms:8.2f} ms {ms / tot:6.3f}  {c:5d} launches  {by / (ms * 1e-3) / 1e9:7.1f} GB/s")

for S in [int(x) for x in args.fc_sessions.split(",") if x]:
    # the FC head over S sessions' features as one batch (chain gesture_fc with S inputs)
    lf = ctx.chain_plan("gesture_features", cfg, 19, n_in)[0]
    fo = m.Ct(torch.empty((2, lf + 1, P.n), dtype=torch.int64, device=dev), lf, 0.0, 0, P.log_n)
    ctx.eval_chain("gesture_features", cfg, ins, m.CtArray([fo]))
    fi = m.CtArray([fo] * S)
    lo = ctx.chain_plan("gesture_fc", cfg, lf, S)
    o_ = m.CtArray([m.Ct(torch.empty((2, l + 1, P.n), dtype=torch.int64, device=dev), l, 0.0, 0, P.log_n) for l in lo])
    ctx.eval_chain("gesture_fc", cfg, fi, o_)
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    ctx.profile()
    ctx.eval_chain("gesture_fc", cfg, fi, o_)
    prof = ctx.profile()
    tot = sum(v[1] for v in prof.values())
    print(f"gesture_fc x {S} sessions: kernel sum {tot:.2f} ms ({tot / S:.3f} ms/session)")
    for k, (c, ms, by, ops) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:16s} {ms:8.2f} ms {ms / tot:6.3f}  {c:5d} launches  {by / (ms * 1e-3) / 1e9:7.1f} GB/s")
