"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel family
launches, total time and share of the library's kernel time.  ncu serialises launches and
runs them cold-cache, so compare shares, not absolute times, with bench.py's profile.
Usage: python tools/launch_summary.py launches.csv [--last-steps-only]"""
import csv
import re
import sys
from collections import defaultdict


def family(name):
    m = re.search(r"mmfhe::\S*?::(\w+)|mmfhe::(\w+)", name)
    if not m:
        return None  # not a library kernel (torch RNG, copies, ...)
    base = m.group(1) or m.group(2)
    if base in ("ntt_fwd_pass", "ntt_inv_pass"):
        # template arguments <LA, LB, COL[, EPI]> (EPI: forward row pass with its epilogue)
        targs = re.search(base + r"<([^>]*)>", name)
        args = [a.strip().replace("(bool)", "").replace("true", "1").replace("false", "0")
                for a in targs.group(1).split(",")] if targs else []
        is_col = len(args) >= 3 and args[2] == "1"
        epi = len(args) >= 4 and args[3] == "1"
        return base.replace("_pass", "_col" if is_col else ("_row_epi" if epi else "_row"))
    return base


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    t = defaultdict(float)
    n = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        f = family(r["Kernel Name"])
        if f is None or f == "mb_kernel":  # microbenchmark: not part of the step
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
        t[f] += v * scale
        n[f] += 1
    tot = sum(t.values())
    print(f"library kernels: {sum(n.values())} launches, {tot / 1e3:.1f} ms (ncu, serialised, cold cache)")
    for f, us in sorted(t.items(), key=lambda kv: -kv[1]):
        print(f"  {f:20s} {n[f]:6d} launches  {us / 1e3:9.2f} ms  share {us / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
