"""Per-step device times of the C2 step (and C4 session) to diagnose run-to-run variance:
python tools/diag_steps.py [n_steps]"""
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
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


def run(tag, sampler=False):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    host = []
    clk = bench.ClockSampler(0) if sampler else None
    if clk:
        clk.__enter__()
    evs[0].record(stream)
    for i in range(n):
        t0 = time.perf_counter()
        for c in ("vitals_v1", "vitals_v2"):
            ctx.eval_chain(c, mcfg, ins_a[c], outs_a[c])
        host.append((time.perf_counter() - t0) * 1e3)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    dev_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
    print(tag, "device ms/step:", [round(x, 1) for x in dev_ms])
    print(tag, "host enqueue ms/step:", [round(x, 1) for x in host])
    print(tag, "pool MB:", ctx.memory() // (1 << 20), "torch MB:", torch.cuda.memory_allocated() // (1 << 20))


for i in range(3):
    for c in ("vitals_v1", "vitals_v2"):
        ctx.eval_chain(c, mcfg, ins_a[c], outs_a[c])
torch.cuda.synchronize()
run("plain")
run("sampler", sampler=True)
run("plain2")

# C4 session, per step
res = []
for i in range(4):
    t0 = time.perf_counter()
    r = bench.bench_workload("C4", m, torch, dev, steps=1, warmup=1 if i == 0 else 0)
    res.append((round(r["ms_per_step"], 1), round(r["kernel_ms_total"], 1), round((time.perf_counter() - t0), 1)))
print("C4 (ms_per_step, kernel_ms, wall_s incl setup):", res)
