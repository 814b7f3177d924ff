"""Per-rank stage times of the N-GPU CCD step, measured on ONE B200.

No 8-GPU node is available, so each rank's device work is run here in turn
exactly as rank r of N would run it (same ccdk calls, same shard ranges),
timed with CUDA events on the context's stream, L2 flushed before each:

  sharded    ccdk_ccd_resident(cfg, r, N): replicated build + sort, the
             SweepRange shard's sweep, its candidates' classify + narrow
  rebalanced ccdk_broad_resident(cfg, r, N) on every rank, then the
             rank-ordered concatenation of all keys is split N ways —
             contiguous equal slices, or interleaved (global index = r mod N,
             multigpu.rebalance_keys' default) — and rank r's share runs
             ccdk_ccd_keys_resident

The predicted N-GPU step is the max over ranks of each phase plus the
collectives (all_gather of N counts, one all_to_all of 8-byte keys, one
8-byte allreduce), estimated from NVLink 5 (~700 GB/s per direction
achieved) and ~15 us per small collective.  Writes one JSON object.

    python tools/predict_scaling.py [--workload C4] [--ns 2,4,8] [--out FILE]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--ns", default="2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from paper_2112_06300_b200 import ccdkit as ck, native, scenes

    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = native.Context(0)
    ctx.set_stream(stream.cuda_stream)
    scene = scenes.config_scene(args.workload)
    cfg = ck.PipelineConfig(inflation=0.01)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    coll_us = 15.0
    nvlink_gbs = 700.0

    def timed(fn):
        best = None
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = fn()
            b.record(stream)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        return best, out

    result = {"workload": args.workload, "primitives": scene.primitive_count(), "per_n": {}}
    with torch.cuda.stream(stream):
        res = ck.ResidentScene(scene, ctx)
        ms1, rep1 = timed(lambda: res.step(cfg))
        result["n1_step_ms"] = ms1
        result["n1_stage_ms"] = {k: rep1.device[k] for k in ("ms_build", "ms_sort", "ms_sweep", "ms_pairsort",
                                                              "ms_classify", "ms_narrow")}
        for n in [int(x) for x in args.ns.split(",")]:
            sharded = []
            for r in range(n):
                ms, rep = timed(lambda r=r: res.step(cfg, r, n))
                sharded.append({"rank": r, "step_ms": ms, "candidates": rep.candidate_count,
                                "sweep_ms": rep.device["ms_sweep"], "narrow_ms": rep.device["ms_narrow"],
                                "prologue_ms": rep.device["ms_build"] + rep.device["ms_sort"]})
            # rebalanced: broad on every rank, then balanced slices of all keys
            broad, keys = [], []
            for r in range(n):
                ms, (cnt, nb, _) = timed(lambda r=r: res.broad(cfg, r, n))
                buf = torch.empty(max(cnt, 1), dtype=torch.int64, device="cuda:0")
                res.copy_keys(buf.data_ptr())
                torch.cuda.synchronize()
                broad.append({"rank": r, "broad_ms": ms, "candidates": cnt})
                keys.append(buf[:cnt].clone())
            allk = torch.cat(keys)
            total = allk.numel()
            narrow = {"contiguous": [], "interleave": []}
            for policy in narrow:
                for r in range(n):
                    if policy == "contiguous":
                        sl = allk[total * r // n:total * (r + 1) // n].contiguous()
                    else:
                        sl = allk[r::n].contiguous()
                    ms, rep = timed(lambda sl=sl: res.narrow_keys(cfg, sl.data_ptr(), sl.numel(), nb))
                    narrow[policy].append({"rank": r, "narrow_step_ms": ms, "queries": rep.query_count,
                                           "generations": rep.device["generations"]})
            moved = {"contiguous": sum(abs(b["candidates"] - total // n) for b in broad) // 2,
                     "interleave": total - total // n}
            exch = {p: 3 * coll_us * 1e-3 + 8.0 * m / (nvlink_gbs * 1e9) * 1e3 for p, m in moved.items()}
            pred = {"sharded": max(x["step_ms"] for x in sharded) + coll_us * 1e-3}
            for policy in narrow:
                pred[f"rebalanced_{policy}"] = (max(b["broad_ms"] for b in broad)
                                                + max(x["narrow_step_ms"] for x in narrow[policy]) + exch[policy])
            result["per_n"][n] = {
                "sharded": sharded, "rebalanced_broad": broad, "rebalanced_narrow": narrow,
                "keys_moved": moved, "collectives_ms_est": exch,
                "predicted_step_ms": pred,
                "predicted_speedup_vs_n1": {k: ms1 / v for k, v in pred.items()},
            }
    txt = json.dumps(result, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
