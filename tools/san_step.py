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
