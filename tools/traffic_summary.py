"""Per-stage DRAM traffic and kernel time of one CCD step from an ncu launch
list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
second of two steps).  Writes the summary text and profiles/traffic_r02.json
entries the bench line's roofline_build / roofline_sort / roofline_pairsort
quote as `traffic`.

    python tools/traffic_summary.py gpurun_out/launches_dram_C4.csv profiles/r02_launches_dram_C4.txt
"""
import collections
import csv
import json
import os
import sys

# stage of each launch, by the step's launch order: K1 | K2+K3 (axis, key
# build, radix sort, permute + quantise) | K4+K5 (slab set-up or run ends,
# heavy segments, sweep) | K6 pair sort | the rest (classify, narrow)
def stage_of(seq):
    stage, out = "other", []
    for n in seq:
        if n == "k_build_boxes":
            stage = "build"
        elif n == "k_axis_sum":
            stage = "sort"
        elif n in ("k_slab_stats", "k_run_ends"):
            stage = "sweep"
        elif stage == "sweep" and "policy_hub<unsigned long long" in n and "Radix" in n:
            stage = "pairsort"
        elif n in ("k_classify_keys", "k_init_scalars"):
            stage = "other"
        out.append(stage)
    return out


def main(path, out_txt):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    data = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = data.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].replace("ccdk::<unnamed>::", "")})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(data)
    second = [data[i] for i in ids if i >= ids[len(ids) // 2]]
    for d, st in zip(second, stage_of([d["name"] for d in second])):
        d["stage"] = st
    agg = collections.OrderedDict()
    for d in second:
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d["gpu__time_duration.sum"] / 1e3
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot_t = sum(a[1] for a in agg.values())
    lines = [f"# {path}: second of two C4 steps, ncu serialised, caches flushed per kernel; total {tot_t:.1f} us",
             f"{'us':>9} {'share':>6} {'n':>4} {'DRAM MB':>9} {'GB/s':>7}  kernel"]
    for name, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:9.1f} {100 * t / tot_t:5.1f}% {n:4d} {b / 1e6:9.2f} {b / 1e3 / t if t else 0:7.0f}  {name[:110]}")
    stage = {}
    for s in ("build", "sort", "sweep", "pairsort"):
        t = sum(d["gpu__time_duration.sum"] / 1e3 for d in second if d["stage"] == s)
        b = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in second if d["stage"] == s)
        stage[s] = (t, b)
        lines.append(f"# stage {s}: {t:.1f} us kernel time, {b / 1e6:.2f} MB DRAM, {b / 1e3 / t if t else 0:.0f} GB/s")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tj = os.path.join(os.path.dirname(os.path.abspath(out_txt)), "traffic_r02.json")
    prev = json.load(open(tj)) if os.path.exists(tj) else {}
    prev.update({f"{s}_bytes_per_step": int(b) for s, (t, b) in stage.items()})
    prev.update({f"{s}_kernel_us_ncu": round(t, 1) for s, (t, b) in stage.items()})
    prev["r02_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum summed over the stage's kernels of one C4 step "
                        f"({os.path.basename(out_txt)}; ncu flushes caches before every kernel, so these are "
                        f"cold-cache bytes)")
    json.dump(prev, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
