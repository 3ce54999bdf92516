"""Summarise an ncu report (or a launch-list CSV) into the text kept under profiles/.

    python scripts/summarize_ncu.py gpurun_out/x.ncu-rep  > profiles/r01/x.txt
    python scripts/summarize_ncu.py --launches gpurun_out/launches.csv > profiles/r01/launches.txt
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(rep):
    h, units, data = raw(rep)
    name_i = h.index("Kernel Name")
    for r in data:
        print(f"kernel: {r[name_i]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:80s} {r[i]:>16s} {units[i]}")
        stalls = [(float(r[i] or 0), n) for i, n in enumerate(h)
                  if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
                  and r[i] not in ("", "n/a")]
        tot = sum(x for x, _ in stalls) or 1.0
        print("  warp-state samples (top):")
        for x, n in sorted(stalls, reverse=True)[:8]:
            print(f"    {100 * x / tot:5.1f}%  {n.replace('smsp__pcsamp_warps_issue_stalled_', '')}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for k, v in agg.items() if "lf::" in k)
    print(f"{'launches':>8} {'mean ns':>12} {'share of lf:: time':>18}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / total:.1f}%" if "lf::" in k and total else "-"
        print(f"{len(v):8d} {sum(v) / len(v):12.0f} {share:>18}  {k[:110]}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1])
