import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, numpy as np
import bench
from paper_2603_22437_b200 import mmfhe as m

dev = torch.device("cuda", 0)
P, cfg = bench.c2_config()
ctx, gen = bench.make_ctx_c2(m, torch, P, cfg, dev, seed=5)
mcfg = bench.chain_cfg_c2(m, cfg)
ins = bench.session_inputs(m, torch, gen, P, cfg, dev)
outs = {c: bench.outputs_for(m, torch, ctx, P, mcfg, c, ins[c], dev) for c in ins}
ctx.trace_enable(False)
for _ in range(3):
    for c in ins:
        ctx.eval_chain(c, mcfg, ins[c], outs[c])
torch.cuda.synchronize()
for c in ins:
    t0 = time.perf_counter()
    ctx.eval_chain(c, mcfg, ins[c], outs[c])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{c}: host enqueue {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms")
ctx.profile_enable(True)
for c in ins:
    ctx.eval_chain(c, mcfg, ins[c], outs[c])
    prof = ctx.profile()
    tot = sum(v[1] for v in prof.values())
    print(c, f"kernel sum {tot:.1f} ms", {k: round(v[1], 2) for k, v in prof.items()})
