"""C2 probe: per-chain device time of the bench's C2 step (vitals_v1 and vitals_v2 timed
separately with CUDA events, graph replay after warm-up) and the top kernels of each.
Usage: python tools/c2probe.py"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402

dev = torch.device("cuda", 0)
P, cfg = bench.c2_config()
ctx, gen = bench.make_ctx_c2(m, torch, P, cfg, dev, seed=5)
mcfg = bench.chain_cfg_c2(m, cfg)
ins = bench.session_inputs(m, torch, gen, P, cfg, dev)
outs = {c: bench.outputs_for(m, torch, ctx, P, mcfg, c, ins[c], dev) for c in ins}
ins_a = {c: m.CtArray(ins[c]) for c in ins}
outs_a = {c: m.CtArray(outs[c]) for c in outs}
ctx.trace_enable(False)
stream = torch.cuda.current_stream(dev)
for c in ins:
    for _ in range(3):
        ctx.eval_chain(c, mcfg, ins_a[c], outs_a[c])
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        ctx.eval_chain(c, mcfg, ins_a[c], outs_a[c])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / 5
    l0 = ctx.launch_count()
    ctx.profile_enable(True)
    ctx.eval_chain(c, mcfg, ins_a[c], outs_a[c])
    prof = ctx.profile()
    ctx.profile_enable(False)
    tot = sum(v[1] for v in prof.values())
    print(f"{c}: {ms:.2f} ms/step (graph replay); profiled kernel sum {tot:.2f} ms, "
          f"{ctx.launch_count() - l0} launches")
    print("   ", {k: round(v[1], 2) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]})
