import sys; sys.path.insert(0, ".")
import torch, bench
from paper_2603_22437_b200 import mmfhe as m
dev = torch.device("cuda", 0)
P, cfg = bench.c2_config()
ctx, gen = bench.make_ctx_c2(m, torch, P, cfg, dev, seed=5)
mcfg = bench.chain_cfg_c2(m, cfg)
ins = bench.session_inputs(m, torch, gen, P, cfg, dev)
outs = {c: bench.outputs_for(m, torch, ctx, P, mcfg, c, ins[c], dev) for c in ins}
ctx.trace_enable(False)
for _ in range(2):
    for c in ins:
        ctx.eval_chain(c, mcfg, ins[c], outs[c])
ctx.profile_enable(True)
for c in ins:
    ctx.eval_chain(c, mcfg, ins[c], outs[c])
prof = ctx.profile()
print({k: round(v[1], 2) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:6]})
