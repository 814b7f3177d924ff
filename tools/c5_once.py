"""One C5 narrow-only batch (device-resident queries), for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_06300_b200 import ccdkit as ck, scenes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
qb = scenes.config_queries(n)
k = torch.from_numpy(qb.kind).cuda()
p = torch.from_numpy(qb.points).cuda()
out = ck.narrow_phase_device(k.data_ptr(), p.data_ptr(), n)
print("C5", n, "device_ms", round(out.device_ms, 3), "evals", out.evaluations, "gens", out.generations)
