"""Step-by-step GPU smoke with progress prints (debug aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
T0 = time.time()
def log(*a):
    print(f"[{time.time()-T0:7.2f}s]", *a, flush=True)
from paper_2112_06300_b200 import ccdkit as ck, scenes, abi, native
log("import ok")
ctx = native.default_context(); log("ctx ok")
d, u = ck.round_reduced(np.array([0.1, 1.0]), ctx); log("round", d.view(np.uint32), u.view(np.uint32))
s = scenes.make_cloth_scene(8, 8, 0.02, 1.0, 1)
b = ck.build_boxes(s, 0.01, ctx=ctx); log("boxes", len(b))
log("axis", ck.choose_axis(b, ctx))
pairs = ck.stq(b, s, ctx=ctx); log("stq pairs", len(pairs))
q = scenes.random_queries(4, seed=1003)
out = ck.narrow_phase(q, ctx=ctx); log("narrow", out.toi, out.total_splits, out.generations)
q = scenes.random_queries(256, seed=1003)
out = ck.narrow_phase(q, ctx=ctx); log("narrow256", out.global_toi, out.total_splits, out.generations)
r = ck.ccd(s, ck.PipelineConfig(inflation=0.01), ctx=ctx); log("ccd", r.toi.toi, r.candidate_count)
import oracle
e, pe = oracle.orc().ccd(s, ck.PipelineConfig(inflation=0.01).to_c()); log("orc", e.toi, e.candidate_count, np.array_equal(pe, r.candidates))
