"""Summarise ncu outputs (launch list CSV and --set full reports) as text for profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches_C4.csv
    python tools/ncu_summary.py report gpurun_out/prof_gen_C4.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    data = rows[hi + 1:]
    ids = sorted({int(r[ii]) for r in data})
    half = ids[len(ids) // 2] if len(sys.argv) < 4 else 0
    agg, cnt, tot = collections.OrderedDict(), collections.Counter(), 0.0
    for r in data:
        if int(r[ii]) < half:
            continue
        name = r[ki].split("(")[0].replace("ccdk::<unnamed>::", "")
        name = name.split("<")[0] if name.startswith("void cub") else name
        v = float(r[vi].replace(",", ""))
        agg[name] = agg.get(name, 0) + v
        cnt[name] += 1
        tot += v
    print(f"# launch list (second of two steps; ncu cold-cache serialised; total {tot / 1e6:.3f} ms)")
    print(f"{'ms':>9} {'share':>6} {'n':>5}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:9.3f} {100 * v / tot:5.1f}% {cnt[k]:5d}  {k}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"# {path}: {name.split('(')[0]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:80s} {row[i]:>18s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
