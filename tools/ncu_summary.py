"""Summarise an ncu report: per-kernel time, DRAM bytes, pipe utilisation, top stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv, io, subprocess, sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__average_warp_latency_issue_stalled_barrier.ratio",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
           "smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio",
           "smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio",
           "smsp__average_warp_latency_issue_stalled_wait.ratio",
           "smsp__average_warp_latency_issue_stalled_mio_throttle.ratio",
           "smsp__average_warp_latency_issue_stalled_lg_throttle.ratio",
           "smsp__average_warp_latency_issue_stalled_not_selected.ratio",
           "smsp__average_warp_latency_issue_stalled_selected.ratio"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].split("::")[-1]
    print(f"== {name}  grid={d.get('launch__grid_size')} block={d.get('launch__block_size')} regs={d.get('launch__registers_per_thread')}")
    for m in METRICS[:10]:
        if m in d:
            u = units[hdr.index(m)]
            print(f"   {m:62s} {d[m]:>12s} {u}")
    # warp-state samples (--set full): share of each stall reason
    full = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    frows = list(csv.reader(io.StringIO(full)))
    fd = dict(zip(frows[0], frows[2 + rows.index(r) - 2])) if len(frows) > 2 else {}
    pre = "smsp__pcsamp_warps_issue_stalled_"
    st = {k[len(pre):]: float(v) for k, v in fd.items()
          if k.startswith(pre) and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
    tot = sum(st.values()) or 1.0
    if "smsp__issue_active.avg.pct_of_peak_sustained_active" in fd:
        print(f"   {'smsp__issue_active.avg.pct_of_peak_sustained_active':62s} "
              f"{fd['smsp__issue_active.avg.pct_of_peak_sustained_active']:>12s} %")
    top = sorted(st.items(), key=lambda kv: -kv[1])[:7]
    print("   warp-state samples:", ", ".join(f"{k} {v / tot:.2f}" for k, v in top))
