"""Full-size parity of the BASELINE configs against the unmodified reference
(oracle/_ref, all host cores): C1-C4 full CCD steps (candidates, per-query ToI
and flags, global ToI, tracked peak) and the whole C5 10M-query batch
(per-query ToI / flags, total splits, peak queue).  Test infrastructure: run
on the GPU box, summary lines go to stdout (profiles/r01_full_parity.txt)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2112_06300_b200 import ccdkit as ck, scenes
from paper_2112_06300_b200.ccdkit import NarrowConfig, PipelineConfig

cores = os.cpu_count() or 1
r = oracle.ref(cores)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


for w in (sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]):
    t0 = time.perf_counter()
    if w == "C5":
        qb = scenes.config_queries(10_000_000)
        got = ck.narrow_phase(qb)
        t1 = time.perf_counter()
        etoi, efl, st = r.narrow_phase(qb.kind, qb.points, NarrowConfig().to_c())
        t2 = time.perf_counter()
        res = {"workload": w, "queries": len(qb),
               "toi_bits_equal": bool(np.array_equal(bits(got.toi), bits(etoi))),
               "flags_equal": bool(np.array_equal(got.flags, efl)),
               "total_splits": [got.total_splits, int(st.total_splits)],
               "peak_queue": [got.peak_queue, int(st.peak_queue)],
               "global_toi": [got.global_toi, float(st.global_toi)],
               "gpu_s": round(t1 - t0, 2), "ref_s": round(t2 - t1, 2), "ref_threads": cores}
    else:
        s = scenes.config_scene(w)
        cfg = PipelineConfig(inflation=0.01)
        rs = ck.ResidentScene(s)
        rep = rs.step(cfg)
        pairs = rs.candidates(rep.candidate_count)
        toi, flags = rs.query_results(rep.query_count)
        t1 = time.perf_counter()
        cref = PipelineConfig(inflation=0.01, broad_method=ck.BROAD_SAP, threads=cores)
        exp, epairs = r.ccd(s, cref.to_c())
        kind, pts, _, _ = r.classify(epairs, s)
        etoi, efl, st = r.narrow_phase(kind, pts, NarrowConfig().to_c())
        t2 = time.perf_counter()
        res = {"workload": w, "primitives": s.nv + s.ne + s.nf,
               "candidates": [rep.candidate_count, int(exp.candidate_count)],
               "candidates_equal": bool(np.array_equal(pairs, epairs)),
               "toi_bits_equal": bool(np.array_equal(bits(toi), bits(etoi))),
               "flags_equal": bool(np.array_equal(flags, efl)),
               "global_toi": [rep.toi.toi, float(exp.toi)],
               "tracked_peak_bytes": [rep.tracked_peak_bytes, int(exp.tracked_peak_bytes)],
               "total_splits": [rep.device.get("total_splits"), int(st.total_splits)],
               "gpu_s": round(t1 - t0, 2), "ref_s": round(t2 - t1, 2), "ref_threads": cores}
    print(json.dumps(res), flush=True)
