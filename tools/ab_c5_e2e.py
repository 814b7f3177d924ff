"""C5 end-to-end through the C ABI from pinned host buffers: wall time, the
narrow phase's own device time, and the raw H2D rate of the box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_06300_b200 import ccdkit as ck, scenes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
qb = scenes.config_queries(n)
kt = torch.from_numpy(qb.kind).pin_memory()
pt = torch.from_numpy(qb.points).pin_memory()
hq = scenes.QueryBatch(kt.numpy(), pt.numpy())
ck.narrow_phase(hq)
torch.cuda.synchronize()
toi_h = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
fl_h = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
for pinned in (False, True, False, True):
    kw = dict(toi_out=toi_h, flags_out=fl_h) if pinned else {}
    t0 = time.perf_counter()
    out = ck.narrow_phase(hq, **kw)
    t1 = time.perf_counter()
    print(f"e2e wall {1e3 * (t1 - t0):.1f} ms (pinned outputs {pinned}), narrow device (sum of chunks) {out.device_ms:.1f} ms")
d = torch.empty(pt.shape, dtype=pt.dtype, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(pt, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"H2D {pt.numel() * 8 / (t1 - t0) / 1e9:.1f} GB/s ({1e3 * (t1 - t0):.1f} ms for {pt.numel() * 8 / 1e9:.2f} GB)")
