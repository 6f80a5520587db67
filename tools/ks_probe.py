"""The evk-streaming key-switch step at N = 2^16 (bench extras.ks_evk_stream): 15 double-hoisted
baby steps of one PS4 ciphertext at the top level (one ModUp, one grouped inner product
k_hoisted_ip_pq streaming the 15 evaluation keys).  The ncu target for the kernel's DRAM bytes.
Usage: python tools/ks_probe.py [reps]"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
from synth.params import ps4  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda", 0)
P = ps4()
ctx = m.Context.from_params(P)
gen = torch.Generator(device=dev)
gen.manual_seed(5)
basis = list(P.q) + list(P.p)
key_shape = (P.dnum(), 2, len(basis))
steps = list(range(1, 16))
for k in steps:
    ctx.load_galois_key(k, bench.uniform_dev(torch, gen, key_shape, basis, P.n, dev))
L = P.L
data = bench.uniform_dev(torch, gen, (2, L + 1), list(P.q), P.n, dev)
a = m.Ct(data, L, float(2 ** P.scale_bits), P.n // 2, P.log_n, m.FORM_EVAL)
buf = torch.empty((15, 2 * (L + 1 + P.K), P.n), dtype=torch.int64, device=dev)
outs = [m.Ct(buf[i], L, 0.0, 0, P.log_n, m.FORM_EVAL, 2) for i in range(15)]
ctx.trace_enable(False)
for _ in range(reps):
    ctx.hrot_hoisted_pq(a, steps, outs)
torch.cuda.synchronize()
evk = P.dnum() * 2 * (L + 1 + P.K) * P.n * 8
print(f"15 PQ baby steps at level {L}: evk bytes {15 * evk}, outputs {15 * 2 * (L + 1 + P.K) * P.n * 8}")
