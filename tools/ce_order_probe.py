"""Probe: does a compute-stream wait on a copy-stream event fire when ITS copy
completes, or only when a later copy queued on the same copy stream completes?"""
import torch, time
n = 667 * 2**20 // 8
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
x = torch.zeros(1024, device="cuda")
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
for variant in ["split-event-then-copy", "copy-copy"]:
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); eA = torch.cuda.Event(enable_timing=True)
        eB = torch.cuda.Event(enable_timing=True); eK = torch.cuda.Event(enable_timing=True)
        t0.record(cs)
        ks.wait_event(t0)
        with torch.cuda.stream(cs):
            d[0].copy_(h[0], non_blocking=True)
            eA.record(cs)
            if variant == "split-event-then-copy":
                torch.cuda._sleep(1000)  # tiny gap kernel on the copy stream
            d[1].copy_(h[1], non_blocking=True)
            eB.record(cs)
        ks.wait_event(eA)
        with torch.cuda.stream(ks):
            x.add_(1)
            eK.record(ks)
        torch.cuda.synchronize()
        print(variant, "A done %.2f ms, B done %.2f ms, kernel after A at %.2f ms" %
              (t0.elapsed_time(eA), t0.elapsed_time(eB), t0.elapsed_time(eK)))
