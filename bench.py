#!/usr/bin/env python
"""Benchmark: the full conservative CCD step on BASELINE.json's ~1M-primitive
scene (C4), device-timed on N GPUs, plus the end-to-end call through the
C ABI and the reference CPU implementation timed on the host cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

One JSON line on rank 0.  `value` = device ms of the whole CCD step (box
build -> STQ broad phase -> classify -> narrow phase -> global min-ToI incl.
the allreduce(min) across ranks), max over ranks; inputs resident in HBM; L2
flushed (256 MiB memset) before every timed step.  `e2e` = the same step
through the C ABI from pinned host buffers (scene H2D, step, report D2H).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CCD step ms + narrow-phase queries/s at 1/2/4/8 B200 vs CPU ref (cores stated)"
WORKLOADS = {
    "C4": "armadillo-rollers-like ~1M primitives: make_cloth_scene(410,410,jitter .02,drop 1,seed 4) "
          "= 1,005,334 boxes; inflation 0.01, delta 1e-6, min_sep 0, max_splits 2^20, t_max 1",
    "C1": "cloth-on-sphere 100x100 + icosphere, seed 1",
    "C2": "cloth-ball-like 224x224 pleated self-contact + ball, seed 2",
    "C3": "n-body-like box soup 13200 + 1% 20x bodies + walls, seed 3",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rebalance", choices=["auto", "on", "off"], default="auto",
                    help="multi-GPU candidate exchange (interleaved, one all_to_all) before the narrow phase "
                         "(auto: off — the slab-mode SweepRange shards balance C4 on their own)")
    ap.add_argument("--c5-queries", type=int, default=10_000_000,
                    help="narrow-phase-only leg (BASELINE config 5); 0 disables")
    ap.add_argument("--c5-steps", type=int, default=3)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region through
    in-process NVML (initialised before the timed region, so sampling is one
    cheap driver query every `period` s; spawning nvidia-smi inside the timed
    region stalls the driver and was measured to distort the step time)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int, period: float | None = None):
        self.index = index
        self.period = period if period is not None else float(os.environ.get("BENCH_CLOCK_PERIOD", "0.1"))
        self.samples = []
        self.sm_max = None
        self.nv = None
        if os.environ.get("BENCH_NO_CLOCKS"):
            return
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.sm_max = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.nv = nv
            for _ in range(3):  # first queries are slow (driver-side setup): keep them out
                self._sample()
            self.samples.clear()
            self.call_ms = 0.0
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        t0 = time.perf_counter()
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, r))
        self.call_ms = max(getattr(self, "call_ms", 0.0), (time.perf_counter() - t0) * 1e3)

    def _run(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self.stop.wait(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.stop = threading.Event()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": [], "samples": 0,
                    "source": "nvml" if self.nv else "unavailable"}
        sm = sorted(s for s, _ in self.samples)
        reasons = set()
        for _, r in self.samples:
            for name, const in self.REASONS:
                bit = getattr(self.nv, const, 0)
                if bit and (r & bit):
                    reasons.add(name)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.sm_max, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml", "period_s": self.period,
                "max_query_ms": round(getattr(self, "call_ms", 0.0), 3)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def measure_fp64_peak():
    """fp64 roofline denominator measured on this box before the timed region:
    dependent-free DADD throughput over every SM (tools/ubench_fp64 --peak;
    MEASURED_PEAKS.json carries only HBM and bf16).  None if unavailable."""
    import subprocess
    exe = os.path.join(ROOT, "tools", "ubench_fp64")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe, "--peak"], capture_output=True, text=True, timeout=60)
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else None
    except Exception:
        return None


def load_traffic():
    """ncu dram byte counts per launch / per step (profiles/traffic_r0N.json,
    newest round first)."""
    out = {}
    for name in ("traffic_r01.json", "traffic_r02.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                out.update(json.load(f))
        except Exception:
            pass
    return out


def bench_config(workload, primitives):
    """The `config` object of BOTH arms (identical keys and values, so the
    driver can match the reference line to ours)."""
    return {"workload": workload, "scene": WORKLOADS[workload], "primitives": primitives,
            "l2": "ours: flushed (256 MiB memset) before every timed step; reference: CPU"}


def host_info():
    """CPU model and the compiler the reference CPU build used (BASELINE.md §2 'Host')."""
    import subprocess
    model = platform.processor() or platform.machine()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cc = subprocess.run(["g++", "-dumpfullversion"], capture_output=True, text=True, timeout=10).stdout.strip()
        compiler = f"g++ {cc} -std=gnu++20 -O3 -DNDEBUG (oracle/Makefile, unmodified reference sources)"
    except Exception:
        compiler = "g++ -O3 (oracle/Makefile)"
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "compiler": compiler}


def cpu_reference_step(scene, cfg_c, threads):
    import oracle
    t0 = time.perf_counter()
    rep, _ = oracle.ref(threads).ccd(scene, cfg_c, want_pairs=False)
    return (time.perf_counter() - t0) * 1e3, rep


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2112_06300_b200 import ccdkit as ck, scenes
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libccdref.so not built"}))
        return 0
    threads = os.cpu_count() or 1
    scene = scenes.config_scene(args.workload)
    cfg = ck.PipelineConfig(inflation=0.01, broad_method=ck.BROAD_SAP, threads=threads)
    times, rep = [], None
    for i in range(args.warmup + args.steps):
        ms, rep = cpu_reference_step(scene, cfg.to_c(), threads)
        if i >= args.warmup:
            times.append(ms)
    ms = sum(times) / len(times)
    sample = (f"full {args.workload} step via ccdkit_ref::ccd (unmodified reference, BroadMethod::SAP "
              f"= identical candidate set to STQ, threads={threads})")
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.workload, scene.primitive_count()),
        "narrow_queries_per_s": rep.query_count / rep.t_np if rep.t_np > 0 else None,
        "candidates": rep.candidate_count, "toi": rep.toi,
        "stage_s": {"CB": rep.t_cb, "BP": rep.t_bp, "SO/CD": rep.t_socd, "NP": rep.t_np},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": threads, "kind": "reference",
                         "sample": sample, **host_info()},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def candidate_fingerprint(pairs):
    """FNV-1a over the (left, right) packed ids in order, as libccdkit_bench computes it."""
    x = 1469598103934665603
    m = (1 << 64) - 1
    for v in pairs.reshape(-1).tolist():
        x = ((x ^ v) * 1099511628211) & m
    return x


def dropin_e2e(args, torch, scene, flush, resident_fp, rep):
    """The reference's own entry point through the drop-in library: one
    ccdkit::ccd(SceneStep, PipelineConfig) call per step (libccdkit.so over the
    C ABI), scene in pageable std::vectors (H2D inside), CcdReport returned by
    value with all candidate pairs (D2H + container fill inside).  Host wall
    time of the synchronous call; L2 flushed before each call."""
    import ctypes as C
    import numpy as np
    lib = C.CDLL(os.path.join(ROOT, "paper_2112_06300_b200", "lib", "libccdkit_bench.so"))
    lib.ccdkit_bench_prepare.restype = C.c_void_p
    lib.ccdkit_bench_prepare.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                         C.c_void_p, C.c_uint64, C.c_double]
    lib.ccdkit_bench_run.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    lib.ccdkit_bench_free.argtypes = [C.c_void_p]
    lib.ccdkit_bench_last_error.restype = C.c_char_p
    arrs = [np.ascontiguousarray(a) for a in (scene.vertices_t0, scene.vertices_t1, scene.edges, scene.faces)]
    h = lib.ccdkit_bench_prepare(arrs[0].ctypes.data, arrs[1].ctypes.data, scene.nv, arrs[2].ctypes.data,
                                 scene.ne, arrs[3].ctypes.data, scene.nf, 0.01)
    ms, ncand, toi, fp = C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()
    times = []
    try:
        for i in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if lib.ccdkit_bench_run(h, C.byref(ms), C.byref(ncand), C.byref(toi), C.byref(fp)) != 0:
                raise RuntimeError(lib.ccdkit_bench_last_error().decode())
            if i >= args.warmup:
                times.append(ms.value)
    finally:
        lib.ccdkit_bench_free(h)
    e2e = sum(times) / len(times)
    return {"value": e2e, "unit": "ms", "h2d_bytes_per_step": int(scene.nbytes),
            "d2h_bytes_per_step": int(16 * ncand.value + C_REPORT_BYTES),
            "api": "ccdkit::ccd(const SceneStep&, const PipelineConfig&) -> CcdReport (libccdkit.so, "
                   "include/ccdkit/pipeline.hpp), pageable host vectors in, all candidates out",
            "timer": "host wall clock around the synchronous call, L2 flushed before each",
            "candidates": int(ncand.value), "toi": toi.value,
            "matches_device_resident_run": bool(ncand.value == rep.candidate_count and toi.value == rep.toi.toi
                                                and (resident_fp is None or fp.value == resident_fp)),
            "steps_ms": [round(t, 3) for t in times]}


def narrow_only_leg(args, torch, ck, scenes, stream, flush, rank, world, local):
    """BASELINE config 5: narrow phase only over 10M mixed VF/EE queries incl.
    rotated near-degenerates and 16 budget-exhausting slides.  Queries are
    sharded by count (contiguous blocks) across ranks; the global ToI is one
    allreduce(min).  Device-timed with queries resident in HBM; e2e through
    the C ABI from pinned host buffers (H2D of the queries, D2H of per-query
    ToI + flags)."""
    import numpy as np
    dev = f"cuda:{local}"
    n_all = args.c5_queries
    qb = scenes.config_queries(n_all)
    lo, hi = rank * n_all // world, (rank + 1) * n_all // world
    n = hi - lo
    kind_h = torch.from_numpy(np.ascontiguousarray(qb.kind[lo:hi])).pin_memory()
    pts_h = torch.from_numpy(np.ascontiguousarray(qb.points[lo:hi])).pin_memory()
    kind_d = kind_h.to(dev)
    pts_d = pts_h.to(dev)
    toi_d = torch.empty(n, dtype=torch.float64, device=dev)
    flags_d = torch.empty(n, dtype=torch.uint8, device=dev)
    gtoi = torch.full((1,), float("inf"), dtype=torch.float64, device=dev)

    def run():
        return ck.narrow_phase_device(kind_d.data_ptr(), pts_d.data_ptr(), n, toi_ptr=toi_d.data_ptr(),
                                      flags_ptr=flags_d.data_ptr())

    with torch.cuda.stream(stream):
        out = run()  # warm-up
        evs = []
        for _ in range(args.c5_steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = run()
            gtoi.fill_(out.global_toi)
            if world > 1:
                torch.distributed.all_reduce(gtoi, op=torch.distributed.ReduceOp.MIN)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        ms = sum(step_ms) / len(step_ms)
        # e2e: host queries -> C ABI -> host per-query results
        e2e_ms = None
        if not args.no_e2e:
            hq = scenes.QueryBatch(kind_h.numpy(), pts_h.numpy())
            # per-query results land in pinned host buffers (the C ABI's
            # caller-provided outputs), allocated outside the timed call
            toi_h = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
            flags_h = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
            ck.narrow_phase(hq, toi_out=toi_h, flags_out=flags_h)  # warm-up: device buffers sized
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = ck.narrow_phase(hq, toi_out=toi_h, flags_out=flags_h)
            b.record(stream)
            torch.cuda.synchronize()
            e2e_ms = a.elapsed_time(b)
    vals = torch.tensor([ms, e2e_ms or 0.0], dtype=torch.float64, device=dev)
    work = torch.tensor([out.evaluations, out.split_actions, out.total_splits], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(work, op=torch.distributed.ReduceOp.SUM)
    ms, e2e_ms = vals.tolist()[0], (vals.tolist()[1] or None)
    evals, splits, total_splits = (int(x) for x in work.tolist())
    leg = {"workload": "C5", "queries": n_all, "data": scenes.CONFIGS["C5"],
           "ms": ms, "queries_per_s": n_all / (ms * 1e-3),
           "global_toi": float(gtoi.item()), "evaluations": evals, "split_actions": splits,
           "total_splits": total_splits, "generations_rank0": out.generations,
           "ms_steps_rank0": [round(x, 3) for x in step_ms],
           "ms_device_runs_rank0": round(out.device_ms, 3),
           "sharding": f"contiguous query blocks x{world}, allreduce(min)",
           "e2e": None if e2e_ms is None else {
               "value": n_all / (e2e_ms * 1e-3), "unit": "queries/s", "ms": e2e_ms,
               "h2d_bytes_per_step": int(kind_h.numel() + pts_h.numel() * 8) * world,
               "d2h_bytes_per_step": 9 * n_all}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.ref_available():
                threads = os.cpu_count() or 1
                m = min(50_000, n_all)
                import time as _t
                t0 = _t.perf_counter()
                ctoi, cfl, cst = oracle.ref(threads).narrow_phase(qb.kind[:m], qb.points[:m],
                                                                  ck.NarrowConfig().to_c())
                cpu_s = _t.perf_counter() - t0
                leg["cpu_baseline"] = {
                    "value": m / cpu_s, "unit": "queries/s", "cores": threads, "kind": "reference",
                    "sample": f"first {m} C5 queries (incl. {m // 10000} rotated near-degenerates, no "
                              f"budget-exhausting ones) via ccdkit_ref::narrow_phase threads={threads}",
                    "bit_exact_vs_gpu": bool(np.array_equal(ctoi.view(np.uint64), toi_d[:m].cpu().numpy().view(np.uint64))
                                             and np.array_equal(cfl, flags_d[:m].cpu().numpy()))}
        except Exception as e:
            leg["cpu_baseline"] = {"error": str(e)}
    return leg


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if distributed:
        import torch.distributed as dist
        if world > 1:  # NCCL's INIT lines (nRanks, transports) go to stderr for the record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2112_06300_b200 import abi, ccdkit as ck, native, scenes
    from paper_2112_06300_b200.multigpu import RebalancedCcd, ShardedCcd
    # auto = the SweepRange shards alone: with the slab-mode sweep each rank's
    # entry-row shard carries a balanced share of narrow work on this scene
    # (profiles/r02_predict_scaling_C4.json: N = 8 step 2.63 ms sharded vs
    # 2.70 ms interleaved, before the rebalance's extra host round trips,
    # measured +0.6 ms at N = 1); --rebalance on exchanges candidates for
    # skewed scenes
    rebalance = args.rebalance == "on"
    Step = RebalancedCcd if rebalance else ShardedCcd

    stream = torch.cuda.Stream()
    ctx = native.Context(local)
    ctx.set_stream(stream.cuda_stream)
    scene = scenes.config_scene(args.workload)
    cfg = ck.PipelineConfig(inflation=0.01)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    clocks = ClockSampler(local)  # NVML initialised outside the timed region
    fp64_measured = measure_fp64_peak() if rank == 0 else None

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    with torch.cuda.stream(stream):
        resident = ck.ResidentScene(scene, ctx)
        sharded = Step(resident, rank, world)
        for _ in range(args.warmup):
            flush.zero_()
            rep = sharded.step(cfg)
        # ---- device-timed region: K full steps, L2 flushed before each
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        with clocks:
            reps = []
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                reps.append(sharded.step(cfg))
                ev[i][1].record(stream)
            torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - t_wall
        dev_ms = [a.elapsed_time(b) for a, b in ev]
        my_ms = sum(dev_ms) / len(dev_ms)
        rep = reps[-1]
        gtoi = sharded.global_toi(rep)

        # ---- e2e through the resident multi-GPU API from pinned host buffers
        e2e_ms = None
        h2d = scene.nbytes
        d2h = C_REPORT_BYTES + 8
        if not args.no_e2e:
            pin = {}
            for name in ("vertices_t0", "vertices_t1", "edges", "faces"):
                a = getattr(scene, name)
                t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.uint32: torch.int32}[a.dtype.type],
                                pin_memory=True)
                tn = t.numpy().view(a.dtype)
                tn[...] = a
                pin[name] = tn
            pscene = scenes.SceneStep(pin["vertices_t0"], pin["vertices_t1"], pin["edges"], pin["faces"])
            e2e_ev = []
            for i in range(args.warmup + args.steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                res = ck.ResidentScene(pscene, ctx)          # H2D + validation
                sh = Step(res, rank, world)
                r = sh.step(cfg)                               # step + report D2H
                sh.global_toi(r)                               # global ToI D2H
                b.record(stream)
                if i >= args.warmup:
                    e2e_ev.append((a, b))
            torch.cuda.synchronize()
            e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev) / len(e2e_ev)
        resident_fp = None
        if world == 1:
            resident_fp = candidate_fingerprint(resident.candidates(rep.candidate_count))

    # ---- e2e through the drop-in: ccdkit::ccd (libccdkit.so) from pageable
    # SceneStep vectors, CcdReport with every candidate pair (pipeline.cpp:218-232)
    dropin = None
    if world == 1 and not args.no_e2e:
        dropin = dropin_e2e(args, torch, scene, flush, resident_fp, rep)

    # ---- max over ranks
    vals = torch.tensor([my_ms, e2e_ms or 0.0, rep.device["ms_narrow"]], dtype=torch.float64,
                        device=f"cuda:{local}")
    counts = torch.tensor([rep.query_count, rep.candidate_count], dtype=torch.float64,
                          device=f"cuda:{local}")
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(counts, op=torch.distributed.ReduceOp.SUM)
    ms, e2e_max, narrow_ms = vals.tolist()
    queries, candidates = (int(x) for x in counts.tolist())

    c5 = None
    if args.c5_queries > 0:
        c5 = narrow_only_leg(args, torch, ck, scenes, stream, flush, rank, world, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.ref_available():
                threads = os.cpu_count() or 1
                cfg_ref = ck.PipelineConfig(inflation=0.01, broad_method=ck.BROAD_SAP, threads=threads)
                cpu_ms, cpu_rep = cpu_reference_step(scene, cfg_ref.to_c(), threads)
                cpu = {"value": cpu_ms, "unit": "ms", "cores": threads, "kind": "reference",
                       "sample": f"one full {args.workload} step, ccdkit_ref::ccd SAP threads={threads}",
                       **host_info(),
                       "narrow_queries_per_s": cpu_rep.query_count / cpu_rep.t_np if cpu_rep.t_np else None,
                       "toi_matches": cpu_rep.toi == gtoi,
                       "candidates_match": cpu_rep.candidate_count == candidates}
        except Exception as e:  # the baseline must not kill the GPU number
            cpu = {"error": str(e)}

    if rank != 0:
        if distributed:
            torch.distributed.destroy_process_group()
        return 0

    peaks = load_peaks()
    clk = clocks.summary()
    sm_max = clk.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    d = rep.device
    # fp64 roofline of the narrow phase: F = 339 E + 96 S non-FMA fp64 ops
    # (SURVEY §8(d)); peak = 148 SMs x 64 fp64 lanes x clock (nominal, not in
    # MEASURED_PEAKS.json, which has only HBM and bf16)
    flops = 339.0 * d["evaluations"] + 96.0 * d["split_actions"]
    # fp64 peak: MEASURED dependent-free DADD throughput on this B200,
    # 62.7 ops/SM/clk (tools/ubench_fp64.cu, profiles/r01_ubench_fp64.txt; the
    # nominal 64 lanes x 148 SMs); MEASURED_PEAKS.json carries only HBM and bf16
    sm_clk = clk.get("sm_mhz") or sm_max
    if fp64_measured:
        fp64_peak = fp64_measured["dadd_tflops"]
        fp64_src = (f"measured in this run before the timed region: tools/ubench_fp64 --peak, dependent-free DADD "
                    f"over all {fp64_measured['sms']} SMs = {fp64_measured['dadd_tflops']:.2f} T ops/s "
                    f"({fp64_measured['ops_per_sm_clk_at_max']:.1f} ops/SM/clk at the {fp64_measured['max_clock_mhz']} "
                    f"MHz max clock); bound is the fp64 pipe (bit-exact fp64 interval arithmetic, no FMA, no tensor cores)")
    else:
        fp64_peak = 148 * 62.7 * sm_clk * 1e6 / 1e12
        fp64_src = ("fallback: DADD rate 62.7/SM/clk measured in round 1 (profiles/r01_ubench_fp64.txt) x 148 SMs x "
                    "sampled SM clock")
    narrow_tf = flops / (d["ms_narrow"] * 1e-3) / 1e12 if d["ms_narrow"] > 0 else 0.0
    k = scene.primitive_count()
    sweep_bytes = 40.0 * k + 8.0 * rep.candidate_count
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    sweep_gbs = sweep_bytes / (d["ms_sweep"] * 1e-3) / 1e9 if d["ms_sweep"] > 0 else 0.0
    traffic = load_traffic()
    roofline = {"kernel": "k_generation (BFS narrow phase, all generations of one step)",
                "bound": "fp64", "achieved": narrow_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": narrow_tf / fp64_peak, "traffic": traffic.get("k_generation_bytes_per_launch"),
                "traffic_note": traffic.get("k_generation_note", traffic.get("note")),
                "peak_source": fp64_src,
                "algorithmic": f"F = 339*E + 96*S, E={d['evaluations']}, S={d['split_actions']}"}
    roofline_sweep = {"kernel": "K4+K5 sweep stage (slab set-up or run ends, heavy segments, row / short / heavy "
                                "sweep kernels)", "bound": "hbm",
                      "achieved": sweep_gbs, "peak": hbm_peak, "unit": "GB/s",
                      "frac": sweep_gbs / hbm_peak,
                      "traffic": traffic.get("sweep_bytes_per_step", traffic.get("k_sweep_rows_bytes_per_launch")),
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                      "algorithmic": f"B = 40k + 8C, k={k}, C={rep.candidate_count}",
                      "pair_tests": d["pair_tests"],
                      "pair_tests_per_s": d["pair_tests"] / (d["ms_sweep"] * 1e-3) if d["ms_sweep"] else None,
                      "sweep": (f"slab mode: {d['sweep_slabs']} slabs, {d['sweep_entries']} entries (boxes incl. "
                                f"copies in further slabs)") if d.get("sweep_slabs") else "1-D sweep"}
    # HBM-bound prologue stages (north_star: "achieved HBM GB/s for the build,
    # sort and sweep"), algorithmic bytes per SURVEY §8(d) over the device
    # stage time of this step; `traffic` = ncu dram bytes of the same stage
    def hbm_roofline(kernel, nbytes, stage_ms, traffic_key, formula):
        gbs = nbytes / (stage_ms * 1e-3) / 1e9 if stage_ms > 0 else 0.0
        return {"kernel": kernel, "bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": gbs / hbm_peak, "bytes": int(nbytes), "stage_ms": stage_ms,
                "traffic": traffic.get(traffic_key), "algorithmic": formula}
    roofline_build = hbm_roofline(
        "k_build_boxes (K1)", 48.0 * scene.nv + 8.0 * scene.ne + 12.0 * scene.nf + 28.0 * k, d["ms_build"],
        "build_bytes_per_step", f"B = 48nv + 8ne + 12nf + 28k, nv={scene.nv}, ne={scene.ne}, nf={scene.nf}")
    roofline_sort = hbm_roofline(
        "K2 axis + K3 key build, radix sort, permute + quantise", 16.0 * k, d["ms_sort"],
        "sort_bytes_per_step", f"B = 16k (u32 key + u32 value, read + write once), k={k}")
    roofline_pairsort = hbm_roofline(
        "K6 candidate key radix sort", 16.0 * rep.candidate_count, d["ms_pairsort"],
        "pairsort_bytes_per_step", f"B = 16C (u64 key read + write once), C={rep.candidate_count}")
    if c5:
        f5 = 339.0 * c5["evaluations"] + 96.0 * c5["split_actions"]
        a5 = f5 / (c5["ms"] * 1e-3) / 1e12 / world
        c5["roofline"] = {"kernel": "k_generation (C5 narrow phase, all generations)", "bound": "fp64",
                          "achieved": a5, "peak": fp64_peak, "unit": "TFLOP/s", "frac": a5 / fp64_peak,
                          "per": "GPU", "algorithmic": f"F = 339*E + 96*S, E={c5['evaluations']}, "
                                                       f"S={c5['split_actions']}"}
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args.workload, k),
        "parallelism": f"sweep-range shards x{world}"
                       + (", candidates interleaved across ranks (one all_to_all)" if rebalance else "")
                       + ", allreduce(min)",
        "narrow_queries_per_s": queries / (narrow_ms * 1e-3) if narrow_ms > 0 else None,
        "candidates": candidates, "queries": queries, "toi": gtoi,
        "stage_ms": {kk: d[kk] for kk in ("ms_build", "ms_sort", "ms_sweep", "ms_pairsort",
                                           "ms_classify", "ms_narrow", "ms_total")},
        "work": {"pair_tests": d["pair_tests"], "evaluations": d["evaluations"],
                 "split_actions": d["split_actions"], "total_splits": d["total_splits"],
                 "generations": d["generations"], "peak_queue": d["peak_queue"]},
        "e2e": dropin if dropin is not None else
               {"value": e2e_max if e2e_ms is not None else None, "unit": "ms",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "multigpu.RebalancedCcd/ShardedCcd over ResidentScene (pinned host scene in, ToI out)"},
        "e2e_resident": {"value": e2e_max if e2e_ms is not None else None, "unit": "ms",
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "api": "ResidentScene upload (pinned host buffers) + ccdk_ccd_resident step + "
                                "global ToI; candidates stay on the device"},
        "roofline": roofline, "roofline_sweep": roofline_sweep, "roofline_build": roofline_build,
        "roofline_sort": roofline_sort, "roofline_pairsort": roofline_pairsort,
        "cpu_baseline": cpu, "clocks": clk,
        "gpu_launches": int(d["kernel_launches"]) * args.steps,
        "wall_s_timed_region": wall,
        "step_ms": [round(x, 3) for x in dev_ms],
        "narrow_only": c5,
    }
    print(json.dumps(line), flush=True)
    if distributed:
        torch.distributed.destroy_process_group()
    return 0


C_REPORT_BYTES = 0


def main():
    global C_REPORT_BYTES
    args = parse()
    from paper_2112_06300_b200 import abi
    import ctypes
    C_REPORT_BYTES = ctypes.sizeof(abi.Report)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
