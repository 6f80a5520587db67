"""Kernel profile of one batched HRot and HMult at N = 2^16 (PS4, top level, batch 8),
the bench's extras_n16 setup.  Usage: python tools/ps4probe.py"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
from synth.params import ps4  # noqa: E402

dev = torch.device("cuda", 0)
P = ps4()
ctx = m.Context.from_params(P, device=0, stream=torch.cuda.current_stream(dev).cuda_stream)
gen = torch.Generator(device=dev)
gen.manual_seed(4242)
basis = list(P.q) + list(P.p)
key_shape = (P.dnum(), 2, len(basis))
ctx.load_relin_key(bench.uniform_dev(torch, gen, key_shape, basis, P.n, dev))
ctx.load_galois_key(1, bench.uniform_dev(torch, gen, key_shape, basis, P.n, dev))
B, L = 8, P.L
data = bench.uniform_dev(torch, gen, (B, 2, L + 1), list(P.q), P.n, dev)
data2 = bench.uniform_dev(torch, gen, (B, 2, L + 1), list(P.q), P.n, dev)
cts = [m.Ct(data[i], L, 2.0 ** P.scale_bits, P.n // 2, P.log_n, m.FORM_EVAL) for i in range(B)]
cts2 = [m.Ct(data2[i], L, 2.0 ** P.scale_bits, P.n // 2, P.log_n, m.FORM_EVAL) for i in range(B)]
obuf = torch.empty((B, 2, L + 1, P.n), dtype=torch.int64, device=dev)
outs = [m.Ct(obuf[i], L, 0.0, 0, P.log_n, m.FORM_EVAL) for i in range(B)]
ctx.trace_enable(False)
for name, fn in (("hrot", lambda: ctx.hrot_batch(cts, 1, outs)), ("hmult", lambda: ctx.hmult_batch(cts, cts2, outs))):
    fn()
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    ctx.profile()
    fn()
    prof = ctx.profile()
    ctx.profile_enable(False)
    tot = sum(v[1] for v in prof.values())
    print(f"{name}: kernel sum {tot * 1e3 / B:.1f} us/op")
    for k, (c, ms, by, ops) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:14s} {ms * 1e3 / B:7.1f} us/op  {c:3d} launches  {by / (ms * 1e-3) / 1e9:7.1f} GB/s")
