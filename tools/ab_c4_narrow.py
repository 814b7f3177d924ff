"""Narrow phase alone on the C4 step's queries (device-resident), for chunking experiments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2112_06300_b200 import ccdkit as ck, scenes
s = scenes.config_scene(sys.argv[1] if len(sys.argv) > 1 else "C4")
r = oracle.ref(os.cpu_count() or 1)
rep, pairs = r.ccd(s, ck.PipelineConfig(inflation=0.01, broad_method=ck.BROAD_SAP, threads=os.cpu_count()).to_c())
kind, pts, _, _ = r.classify(pairs, s)
k = torch.from_numpy(np.ascontiguousarray(kind)).cuda()
p = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
for i in range(3):
    out = ck.narrow_phase_device(k.data_ptr(), p.data_ptr(), len(kind))
print("chunk", os.environ.get("CCDK_CHUNK", "default"), "n", len(kind), "device_ms", round(out.device_ms, 3), "splits", out.total_splits)
