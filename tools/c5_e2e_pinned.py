"""C5 end to end through ck.narrow_phase from pinned host inputs into pinned host outputs
(the bench's e2e leg), median of 3 wall times."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_06300_b200 import ccdkit as ck, scenes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
qb = scenes.config_queries(n)
kt = torch.from_numpy(qb.kind).pin_memory()
pt = torch.from_numpy(qb.points).pin_memory()
hq = scenes.QueryBatch(kt.numpy(), pt.numpy())
toi_h = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
fl_h = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
ck.narrow_phase(hq, toi_out=toi_h, flags_out=fl_h)
ws, ds = [], []
for _ in range(3):
    t0 = time.perf_counter()
    out = ck.narrow_phase(hq, toi_out=toi_h, flags_out=fl_h)
    ws.append(1e3 * (time.perf_counter() - t0))
    ds.append(out.device_ms)
print(f"first_chunk={os.environ.get('CCDK_FIRST_CHUNK', '1.0')} e2e {statistics.median(ws):.1f} ms, device sum {statistics.median(ds):.1f} ms, toi {out.global_toi}, splits {out.total_splits}")
