"""One warm-up + N device-resident CCD steps on a BASELINE workload (profiling driver)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_06300_b200 import ccdkit as ck, scenes
w = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = scenes.config_scene(w)
rs = ck.ResidentScene(s)
cfg = ck.PipelineConfig(inflation=0.01)
for i in range(1 + n):
    r = rs.step(cfg)
print(w, "toi", r.toi.toi, "cands", r.candidate_count, {k: round(v, 3) for k, v in r.device.items() if k.startswith("ms_")})
