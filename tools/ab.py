"""A/B timing on the GPU box (one parametrised tool; pair with
tools/build_variant.py and CCDK_LIB=... or CCDK_* environment switches).

    python tools/ab.py step [C1..C4] [steps]   device-resident CCD step, median stage ms
    python tools/ab.py c5 [n]                  narrow-only C5 batch, device-resident queries
    python tools/ab.py c5-e2e [n]              C5 from pinned host buffers into pinned outputs
    python tools/ab.py narrow [C1..C4]         narrow phase alone on a step's queries
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def tag():
    return (os.environ.get("CCDK_LIB") or "x/default/x").split("/")[-2]


def step(w="C4", n="10"):
    from paper_2112_06300_b200 import ccdkit as ck, scenes
    rs = ck.ResidentScene(scenes.config_scene(w))
    cfg = ck.PipelineConfig(inflation=0.01)
    reps = [rs.step(cfg) for _ in range(int(n) + 2)][2:]
    med = {k: round(statistics.median(r.device[k] for r in reps), 3) for k in reps[0].device if k.startswith("ms_")}
    r = reps[-1]
    print(tag(), w, "toi", r.toi.toi, "q", r.query_count, "gens", r.device["generations"],
          "splits", r.device["total_splits"], "evals", r.device["evaluations"], med)


def c5(n="10000000"):
    import torch
    from paper_2112_06300_b200 import ccdkit as ck, scenes
    n = int(n)
    qb = scenes.config_queries(n)
    k, p = torch.from_numpy(qb.kind).cuda(), torch.from_numpy(qb.points).cuda()
    for _ in range(3):
        out = ck.narrow_phase_device(k.data_ptr(), p.data_ptr(), n)
    print(tag(), "C5", n, "device_ms", round(out.device_ms, 3), "evals", out.evaluations, "gens", out.generations)


def c5_e2e(n="10000000"):
    import torch
    from paper_2112_06300_b200 import ccdkit as ck, scenes
    n = int(n)
    qb = scenes.config_queries(n)
    hq = scenes.QueryBatch(torch.from_numpy(qb.kind).pin_memory().numpy(),
                           torch.from_numpy(qb.points).pin_memory().numpy())
    toi_h = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    fl_h = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
    ck.narrow_phase(hq, toi_out=toi_h, flags_out=fl_h)
    ws, ds = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        out = ck.narrow_phase(hq, toi_out=toi_h, flags_out=fl_h)
        ws.append(1e3 * (time.perf_counter() - t0))
        ds.append(out.device_ms)
    print(f"{tag()} C5 e2e {statistics.median(ws):.1f} ms, device sum {statistics.median(ds):.1f} ms, "
          f"toi {out.global_toi}, splits {out.total_splits}")


def narrow(w="C4"):
    import torch
    from paper_2112_06300_b200 import ccdkit as ck, scenes
    s = scenes.config_scene(w)
    rep = ck.ccd(s, ck.PipelineConfig(inflation=0.01))
    cq = ck.classify(rep.candidates, s)
    k = torch.from_numpy(cq.queries.kind).cuda()
    p = torch.from_numpy(cq.queries.points).cuda()
    for _ in range(3):
        out = ck.narrow_phase_device(k.data_ptr(), p.data_ptr(), len(cq.queries.kind))
    print(tag(), w, "narrow n", len(cq.queries.kind), "device_ms", round(out.device_ms, 3), "splits", out.total_splits)


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "step"
    {"step": step, "c5": c5, "c5-e2e": c5_e2e, "narrow": narrow}[cmd](*sys.argv[2:])
