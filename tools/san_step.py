"""Small CCD step + narrow phase for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_06300_b200 import ccdkit as ck, scenes
s = scenes.make_cloth_scene(60, 60, 0.02, 1.0, 1)
rs = ck.ResidentScene(s)
r = rs.step(ck.PipelineConfig(inflation=0.01))
print("toi", r.toi.toi, r.candidate_count)
q = scenes.random_queries(3000, seed=1003)
out = ck.narrow_phase(q)
print("narrow", out.total_splits)
# run_batched on a caller's list: shuffled, one owner duplicated, bf halving
import numpy as np
from paper_2112_06300_b200 import abi
b = ck.build_boxes(s, 0.01)
sel = np.random.default_rng(2).permutation(len(b))
sel = np.concatenate([sel, sel[:50]])
boxes = ck.Boxes(b.min_corner[sel], b.max_corner[sel], b.owner_kind[sel], b.owner_index[sel])
for m in (abi.BROAD_STQ, abi.BROAD_BF):
    t = ck.BatchTrace()
    toi = ck.run_batched(s, boxes, ck.PipelineConfig(broad_method=m, memory_budget=1 << 21), t)
    print("run_batched", m, toi.toi, t.broad_batches, t.narrow_batches)
