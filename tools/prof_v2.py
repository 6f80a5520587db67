"""Profiling driver: one C2 vitals_v2 session (F=256, N=2^14) on cuda:0, no warm-up,
so that `ncu -k regex:... -c N` captures the first, representative batched
launches (import NTT, ModUp BConv, ModUp NTT, key inner product, ModDown)."""
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
chain = sys.argv[1] if len(sys.argv) > 1 else "vitals_v2"
outs = bench.outputs_for(m, torch, ctx, P, mcfg, chain, ins[chain], dev)
ctx.trace_enable(False)
ctx.eval_chain(chain, mcfg, ins[chain], outs)
torch.cuda.synchronize()
print("done", chain, ctx.launch_count())
