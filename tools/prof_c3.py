"""Profiling driver: one C3 step (K3 DFT, 32 frames, N=2^15) on cuda:0."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
print(bench.bench_workload(sys.argv[1] if len(sys.argv) > 1 else "C3", m, torch, torch.device("cuda", 0), steps=1, warmup=1))
