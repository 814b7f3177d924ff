"""A/B timing of the device-resident CCD step (median stage ms over N steps).
    CCDK_LIB=... python tools/ab_step.py C4 10"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_06300_b200 import ccdkit as ck, scenes
w = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
s = scenes.config_scene(w)
rs = ck.ResidentScene(s)
cfg = ck.PipelineConfig(inflation=0.01)
reps = [rs.step(cfg) for _ in range(n + 2)][2:]
med = {k: round(statistics.median(r.device[k] for r in reps), 3) for k in reps[0].device if k.startswith("ms_")}
r = reps[-1]
print((os.environ.get("CCDK_LIB") or "x/default/x").split("/")[-2], w, "toi", r.toi.toi, "q", r.query_count, "gens", r.device["generations"], "splits", r.device["total_splits"],
      "evals", r.device["evaluations"], med)
