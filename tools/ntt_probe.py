"""NTT probe: per-pass throughput of the batched forward/inverse NTT at N = 2^13 (PS1),
2^14 (PS2), 2^15 (PS3) and 2^16 (PS4) on cuda:0, against the in-run CT/GS butterfly microbenchmarks.
Usage: python tools/ntt_probe.py [iters]   (also the target for ncu captures)."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_22437_b200 import mmfhe as m  # noqa: E402
from synth.params import ps1, ps2, ps3, ps4  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for P, rows in ((ps1(), 8192), (ps2(), 4096), (ps3(), 2048), (ps4(), 1020)):
    ctx = m.Context.from_params(P)
    primes = list(P.q)
    idx = [i % len(primes) for i in range(rows)]
    qs = torch.tensor([primes[i] for i in idx], dtype=torch.float64, device="cuda:0")
    x = (torch.rand(rows, P.n, dtype=torch.float64, device="cuda:0") * qs[:, None]).to(torch.int64)
    for _ in range(2):
        ctx.ntt(x, idx)
        ctx.ntt(x, idx, inverse=True)
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    ctx.profile()
    for _ in range(iters):
        ctx.ntt(x, idx)
        ctx.ntt(x, idx, inverse=True)
    torch.cuda.synchronize()
    prof = ctx.profile()
    ctx.profile_enable(False)
    ct, gs = ctx.microbench(4), ctx.microbench(5)  # the NTT's own (truncated-quotient) butterflies
    ct0, gs0 = ctx.microbench(0), ctx.microbench(1)
    print(f"log_n={P.log_n} rows={rows}")
    for k in ("ntt_fwd_col", "ntt_fwd_row", "ntt_inv_row", "ntt_inv_col"):
        c, ms, b, ops = prof[k]
        rate = ops / (ms * 1e-3)
        peak = ct if "fwd" in k else gs
        print(f"  {k:12s} {ms / c * 1e3:8.1f} us/launch  {rate / 1e9:7.1f} Gbfly/s  frac {rate / peak:.3f}  "
              f"hbm {b / (ms * 1e-3) / 1e9:7.1f} GB/s")
    print(f"  peaks: CT {ct / 1e9:.1f} GS {gs / 1e9:.1f} Gbfly/s (exact-quotient Shoup: CT {ct0 / 1e9:.1f} "
          f"GS {gs0 / 1e9:.1f})")
    ctx.close()
