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
    st = {m.split('stalled_')[1].split('.')[0]: d[m] for m in METRICS[13:] if m in d}
    print("   stalls(cycles/issue):", st)
