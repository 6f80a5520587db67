"""One forward and one inverse batched NTT at N = 2^16 (PS4 primes, 1040 rows = 52 x 20 limbs)
on cuda:0: the ncu target whose DRAM bytes per launch give profiles/r02/ncu_traffic.json
(algorithmic bytes = one read + one write of every word per pass = 16 B x rows x N).
Usage: python tools/ntt16_probe.py"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
from synth.params import ps4  # noqa: E402

P = ps4()
rows = 1040
ctx = m.Context.from_params(P)
idx = [i % len(P.q) for i in range(rows)]
qs = torch.tensor([P.q[i] for i in idx], dtype=torch.float64, device="cuda:0")
x = (torch.rand(rows, P.n, dtype=torch.float64, device="cuda:0") * qs[:, None]).to(torch.int64)
ctx.ntt(x, idx)
ctx.ntt(x, idx, inverse=True)
torch.cuda.synchronize()
print(f"rows={rows} N={P.n} alg_bytes_per_pass={16 * rows * P.n}")
