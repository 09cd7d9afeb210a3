"""Key counters of an ncu --set full report (one kernel): time, FP64 pipe, issue, occupancy,
registers, DRAM traffic, L1/L2, and the warp-stall split -- the lines profiles/*.txt summaries carry.

usage: python tools/ncu_summary.py REPORT.ncu-rep [label]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print("# %s  kernel %s" % (sys.argv[2] if len(sys.argv) > 2 else rep, name))
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print("%-72s %s %s" % (k, v[i], units[i]))
    # L1 data-pipe wavefronts by kind (shared / global / reductions ...)
    for i, k in enumerate(h):
        if k.startswith("l1tex__data_pipe_lsu_wavefronts") and k.endswith(".sum") and k not in KEYS:
            print("%-72s %s %s" % (k, v[i], units[i]))
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    print("# warp-stall samples: " + ", ".join("%s %.1f%%" % (n, 100 * s / tot) for s, n in sorted(stalls, reverse=True)[:8]))


if __name__ == "__main__":
    main()
