"""Integer microbenchmarks (mmfhe_microbench kinds 0-6) on cuda:0.  Usage: python tools/mb_probe.py"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
from synth.params import ps4  # noqa: E402

ctx = m.Context.from_params(ps4())
names = ["CT bfly", "GS bfly", "MAC128", "Shoup", "CT bfly (lazy4)", "GS bfly (lazy4)"]
for k in range(6):
    v = max(ctx.microbench(k) for _ in range(3))
    print(f"kind {k} {names[k]:18s} {v / 1e9:8.1f} G/s")
