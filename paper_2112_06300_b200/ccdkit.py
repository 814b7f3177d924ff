"""Python mirror of the reference ccdkit API for the CCD hot path.

Same names, argument meaning and error behaviour as the C++ declarations in
proj/include/ccdkit/{aabb,broadphase,narrowphase,pipeline}.hpp; every compute
call goes through the C ABI (include/ccdk.h) to the sm_100a kernels.  The
``threads`` arguments are accepted and ignored (advisory in the reference).

Data types are numpy-level restatements of the reference structs:

* ``Boxes``            vector<Aabb>           (aabb.hpp:20-39)
* pairs (n, 2) u64     vector<CandidatePair>  ids packed (kind << 32) | index
* ``QueryBatch``       vector<NarrowQuery>    (scenes.QueryBatch)
* ``NarrowOutcome``    NarrowOutcome          (narrowphase.hpp:84-90)
* ``CcdReport``        CcdReport              (pipeline.hpp:47-61)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .abi import P_F32, P_F64, P_U8, P_U16, P_U32, P_U64
from .native import (CapacityError, ConfigError, InvalidInput, check, default_context, f32, f64, lib,
                     p, u8, u16, u32, u64)
from .scenes import QueryBatch, SceneStep

__all__ = [
    "Boxes", "SweepRange", "StqStats", "NarrowConfig", "PipelineConfig", "ToiResult",
    "NarrowOutcome", "CcdReport", "InvalidInput", "ConfigError", "CapacityError",
    "round_down_reduced", "round_up_reduced", "round_reduced", "build_boxes", "choose_axis",
    "stq", "bf", "sap", "classify", "inclusion_box", "inclusion_boxes", "process_interval",
    "split_box", "narrow_phase", "ccd", "KIND_VERTEX", "KIND_EDGE", "KIND_FACE", "pack_id",
]

KIND_VERTEX, KIND_EDGE, KIND_FACE = abi.KIND_VERTEX, abi.KIND_EDGE, abi.KIND_FACE
K_NO_COLLISION = float("inf")  # kNoCollision (narrowphase.hpp:41)
K_ZERO_TOI_RETRY_SCALE = 0.8   # pipeline.hpp:87


def pack_id(kind: int, index: int) -> int:
    return (int(kind) << 32) | int(index)


@dataclass
class Boxes:
    min_corner: np.ndarray  # (k, 3) float32
    max_corner: np.ndarray  # (k, 3) float32
    owner_kind: np.ndarray  # (k,) uint8
    owner_index: np.ndarray  # (k,) uint32

    def __len__(self):
        return int(self.min_corner.shape[0])

    def as_tuple(self):
        return self.min_corner, self.max_corner, self.owner_kind, self.owner_index


@dataclass
class SweepRange:
    begin: int = 0
    end: int = abi.UINT64_MAX


@dataclass
class StqStats:
    max_queue: int = 0
    round_sizes: list = field(default_factory=list)
    pair_tests: int = 0
    axis: int = 0
    axis_flags: int = 0  # bit0 near tie under the tree sums, bit1 serial order decided


@dataclass
class NarrowConfig:
    delta: float = 1e-6
    min_separation: float = 0.0
    t_max: float = 1.0
    max_splits: int = 1 << 20
    no_zero_toi: bool = False

    def to_c(self) -> abi.NarrowCfg:
        return abi.narrow_cfg(self.delta, self.min_separation, self.t_max, self.max_splits,
                              self.no_zero_toi)

    def validate(self):
        check(_validate_narrow(self))


def _validate_narrow(c: NarrowConfig) -> int:
    # NarrowConfig::validate (narrowphase.cpp:10-20); mirrored for a clean
    # error before any device work.
    if not (c.delta > 0.0) or c.max_splits < 1 or c.min_separation < 0.0 \
            or not (c.t_max > 0.0) or c.t_max > 1.0:
        raise ConfigError(abi.CONFIG, "NarrowConfig: invalid")
    return abi.OK


BROAD_STQ, BROAD_BF, BROAD_SAP = abi.BROAD_STQ, abi.BROAD_BF, abi.BROAD_SAP
MINSEP_ABSOLUTE, MINSEP_RELATIVE = abi.MINSEP_ABSOLUTE, abi.MINSEP_RELATIVE


@dataclass
class PipelineConfig:
    narrow: NarrowConfig = field(default_factory=NarrowConfig)
    broad_method: int = BROAD_STQ
    memory_budget: int = abi.SIZE_MAX_DIV4
    record_sizes: tuple = (56, 192, 252, 8)
    min_sep_mode: int = MINSEP_ABSOLUTE
    min_sep_fraction: float = 0.2
    threads: int = 1
    inflation: float = 0.0

    def to_c(self) -> abi.PipelineCfg:
        return abi.pipeline_cfg(self.narrow.to_c(), self.broad_method, self.memory_budget,
                                self.min_sep_mode, self.min_sep_fraction, self.threads,
                                self.inflation, self.record_sizes)


@dataclass
class ToiResult:
    toi: float = K_NO_COLLISION
    tolerance_hit: bool = False
    zero_toi_diagnostic: bool = False

    def collision(self) -> bool:
        return self.toi != K_NO_COLLISION


@dataclass
class NarrowOutcome:
    toi: np.ndarray            # per-query ToI (n,) float64
    flags: np.ndarray          # per-query bit0 tolerance_hit, bit1 zero_toi_diagnostic
    global_toi: float
    overflow: bool
    peak_queue: int
    total_splits: int
    evaluations: int = 0
    split_actions: int = 0
    generations: int = 0
    device_ms: float = 0.0

    @property
    def per_query(self):
        return [ToiResult(float(t), bool(f & 1), bool(f & 2)) for t, f in zip(self.toi, self.flags)]


@dataclass
class CcdReport:
    toi: ToiResult
    candidate_count: int
    query_count: int
    batch_count: int
    per_stage_times: dict
    tracked_peak_bytes: int
    candidates: np.ndarray | None
    inflation_policy: str = "per-axis"
    device: dict = field(default_factory=dict)


@dataclass
class BatchTrace:
    """BatchTrace (pipeline.hpp:69-72): batches run_batched actually ran."""
    broad_batches: int = 0
    narrow_batches: int = 0


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# ------------------------------------------------------------------ aabb.hpp

def round_reduced(x, ctx=None):
    """Batched round_down_reduced / round_up_reduced (aabb.hpp:10-14)."""
    x = f64(np.atleast_1d(x))
    dn = np.empty(x.size, np.float32)
    up = np.empty(x.size, np.float32)
    c = _ctx(ctx)
    check(lib().ccdk_round_reduced(c.h, p(x, P_F64), x.size, p(dn, P_F32), p(up, P_F32)))
    return dn, up


def round_down_reduced(x: float, ctx=None) -> np.float32:
    return round_reduced(x, ctx)[0][0]


def round_up_reduced(x: float, ctx=None) -> np.float32:
    return round_reduced(x, ctx)[1][0]


def build_boxes(scene: SceneStep, inflation: float = 0.0, threads: int = 1, ctx=None) -> Boxes:
    """build_boxes (aabb.hpp:49-50): one box per V, E, F in index order."""
    k = scene.primitive_count()
    mn = np.empty((k, 3), np.float32)
    mx = np.empty((k, 3), np.float32)
    kind = np.empty(k, np.uint8)
    idx = np.empty(k, np.uint32)
    c = _ctx(ctx)
    if scene.vertices_t0.shape != scene.vertices_t1.shape:
        raise InvalidInput(abi.INVALID_INPUT, "vertex snapshots differ in length")
    check(lib().ccdk_build_boxes(c.h, p(scene.vertices_t0, P_F64), p(scene.vertices_t1, P_F64),
                                 scene.nv, p(scene.edges, P_U32), scene.ne, p(scene.faces, P_U32),
                                 scene.nf, float(inflation), p(mn, P_F32), p(mx, P_F32),
                                 p(kind, P_U8), p(idx, P_U32)))
    return Boxes(mn, mx, kind, idx)


# ------------------------------------------------------------ broadphase.hpp

def choose_axis(boxes: Boxes, ctx=None) -> int:
    c = _ctx(ctx)
    a = C.c_int()
    mn, mx = f32(boxes.min_corner), f32(boxes.max_corner)
    check(lib().ccdk_choose_axis(c.h, p(mn, P_F32), p(mx, P_F32), len(boxes), C.byref(a)))
    return a.value


def _broad(method, boxes: Boxes, scene: SceneStep, stats, rng, ctx):
    c = _ctx(ctx)
    rng = rng or SweepRange()
    mn, mx = f32(boxes.min_corner), f32(boxes.max_corner)
    kd, ix = u8(boxes.owner_kind), u32(boxes.owner_index)
    n = C.c_uint64()
    st = abi.StqStats()
    with c.lock:  # the pairs and round sizes are the context's until its next call
        check(lib().ccdk_broad_phase(c.h, method, p(mn, P_F32), p(mx, P_F32), p(kd, P_U8), p(ix, P_U32),
                                     len(boxes), scene.nv, p(scene.edges, P_U32), scene.ne,
                                     p(scene.faces, P_U32), scene.nf, rng.begin, rng.end, C.byref(n),
                                     C.byref(st)))
        out = np.empty((n.value, 2), np.uint64)
        if n.value:
            check(lib().ccdk_fetch_pairs(c.h, p(out, P_U64)))
        rounds = np.empty(st.n_rounds if stats is not None else 0, np.uint64)
        if stats is not None and st.n_rounds:
            check(lib().ccdk_fetch_round_sizes(c.h, p(rounds, P_U64)))
    if stats is not None:
        stats.round_sizes.extend(int(x) for x in rounds)
        stats.max_queue = max(stats.max_queue, int(st.max_queue))
        stats.pair_tests = int(st.pair_tests)
        stats.axis = int(st.axis)
        stats.axis_flags = int(st.axis_flags)
    return out


def stq(boxes: Boxes, scene: SceneStep, threads: int = 1, stats: StqStats | None = None,
        range: SweepRange | None = None, ctx=None) -> np.ndarray:  # noqa: A002
    """stq (broadphase.hpp:57-59): canonical candidate pairs (n, 2) u64."""
    return _broad(BROAD_STQ, boxes, scene, stats, range, ctx)


def bf(boxes: Boxes, scene: SceneStep, threads: int = 1, range: SweepRange | None = None,
       ctx=None) -> np.ndarray:  # noqa: A002
    return _broad(BROAD_BF, boxes, scene, None, range, ctx)


def sap(boxes: Boxes, scene: SceneStep, threads: int = 1, range: SweepRange | None = None,
        ctx=None) -> np.ndarray:  # noqa: A002
    return _broad(BROAD_SAP, boxes, scene, None, range, ctx)


@dataclass
class ClassifiedQueries:
    queries: QueryBatch      # VF block then EE block
    sources: np.ndarray      # (n, 2) u64 source pairs
    n_vf: int

    @property
    def vertex_face(self):
        return self.queries.slice(0, self.n_vf)

    @property
    def edge_edge(self):
        return self.queries.slice(self.n_vf, len(self.queries))


def classify(pairs: np.ndarray, scene: SceneStep, ctx=None) -> ClassifiedQueries:
    """classify (broadphase.hpp:78-79)."""
    c = _ctx(ctx)
    pairs = u64(pairs).reshape(-1, 2)
    n = pairs.shape[0]
    kind = np.empty(max(n, 1), np.uint8)
    pts = np.empty((max(n, 1), 24), np.float64)
    src = np.empty((max(n, 1), 2), np.uint64)
    nvf, nee = C.c_uint64(), C.c_uint64()
    check(lib().ccdk_classify(c.h, p(pairs, P_U64), n, p(scene.vertices_t0, P_F64),
                              p(scene.vertices_t1, P_F64), scene.nv, p(scene.edges, P_U32), scene.ne,
                              p(scene.faces, P_U32), scene.nf, p(kind, P_U8), p(pts, P_F64),
                              p(src, P_U64), C.byref(nvf), C.byref(nee)))
    m = nvf.value + nee.value
    return ClassifiedQueries(QueryBatch(kind[:m].copy(), pts[:m].copy()), src[:m].copy(), nvf.value)


# ----------------------------------------------------------- narrowphase.hpp

def inclusion_boxes(kind, points, boxes, ctx=None) -> np.ndarray:
    """Batched inclusion_box (narrowphase.hpp:59): boxes (n, 6) = (tlo, thi,
    ulo, uhi, vlo, vhi) -> (n, 6) = (x.lo, x.hi, y.lo, y.hi, z.lo, z.hi)."""
    c = _ctx(ctx)
    kind = u8(np.atleast_1d(kind))
    points = f64(points).reshape(-1, 24)
    boxes = f64(boxes).reshape(-1, 6)
    out = np.empty((kind.size, 6), np.float64)
    check(lib().ccdk_inclusion_boxes(c.h, p(kind, P_U8), p(points, P_F64), p(boxes, P_F64), kind.size,
                                     p(out, P_F64)))
    return out


def inclusion_box(kind: int, points, box=(0.0, 1.0, 0.0, 1.0, 0.0, 1.0), ctx=None) -> np.ndarray:
    return inclusion_boxes([kind], points, box, ctx)[0]


def process_intervals(kind, points, boxes, depth, t_star, cfg: NarrowConfig, sep=None, ctx=None):
    """Batched process_interval (narrowphase.hpp:77-79).  Returns (action,
    candidate_t, zero_diag, children (n, 12), child_depth (n, 6))."""
    c = _ctx(ctx)
    kind = u8(np.atleast_1d(kind))
    n = kind.size
    points = f64(points).reshape(n, 24)
    boxes = f64(boxes).reshape(n, 6)
    depth = u16(depth).reshape(n, 3)
    t_star = f64(np.broadcast_to(t_star, (n,)))
    sep_a = None if sep is None else f64(np.broadcast_to(sep, (n,)))
    action = np.empty(n, np.uint8)
    ct = np.empty(n, np.float64)
    zd = np.empty(n, np.uint8)
    ch = np.empty((n, 12), np.float64)
    cd = np.empty((n, 6), np.uint16)
    ccfg = cfg.to_c()
    check(lib().ccdk_process_intervals(c.h, p(kind, P_U8), p(points, P_F64), p(boxes, P_F64),
                                       p(depth, P_U16), p(t_star, P_F64), p(sep_a, P_F64), n,
                                       C.byref(ccfg), p(action, P_U8), p(ct, P_F64), p(zd, P_U8),
                                       p(ch, P_F64), p(cd, P_U16)))
    return action, ct, zd, ch, cd


def process_interval(kind, points, box, depth, t_star, cfg: NarrowConfig, min_separation=-1.0,
                     ctx=None):
    a, ct, zd, ch, cd = process_intervals([kind], points, box, depth, t_star, cfg,
                                          sep=min_separation, ctx=ctx)
    return int(a[0]), float(ct[0]), bool(zd[0]), ch[0], cd[0]


def split_box(box, depth, d: int):
    """split_box (narrowphase.cpp:122-132): exact bisection of dimension d.
    Pure index/bit bookkeeping on six doubles (no floating-point search), so
    it is restated on the host like the reference's inline helper."""
    box = np.array(box, np.float64).reshape(6)
    depth = np.array(depth, np.uint16).reshape(3)
    lo, hi = box[2 * d], box[2 * d + 1]
    mid = lo + 0.5 * (hi - lo)
    left, right = box.copy(), box.copy()
    left[2 * d + 1] = mid
    right[2 * d] = mid
    dl = depth.copy()
    dl[d] += 1
    return left, dl, right, dl.copy()


def _out_array(a, n: int, dtype, name: str) -> np.ndarray:
    if a is None:
        return np.empty(max(n, 1), dtype)
    if a.dtype != dtype or a.ndim != 1 or a.shape[0] < n or not a.flags.c_contiguous or not a.flags.writeable:
        raise ConfigError(abi.CONFIG, f"narrow_phase: {name} must be a writable contiguous {np.dtype(dtype)}[{n}]")
    return a if n else np.empty(1, dtype)


def narrow_phase(queries: QueryBatch, cfg: NarrowConfig | None = None, threads: int = 1,
                 queue_capacity: int = abi.UINT64_MAX, per_query_min_sep=None,
                 ctx=None, toi_out=None, flags_out=None) -> NarrowOutcome:
    """narrow_phase (narrowphase.hpp:97-100).  ``toi_out`` / ``flags_out``
    (float64[n] / uint8[n], C-contiguous; e.g. views of pinned host memory)
    receive the per-query results in place, as the C ABI's caller-provided
    output buffers do; by default fresh arrays are returned."""
    cfg = cfg or NarrowConfig()
    c = _ctx(ctx)
    n = len(queries)
    if per_query_min_sep is not None and len(per_query_min_sep) != n:
        raise ConfigError(abi.CONFIG, "narrow_phase: per-query separation list size mismatch")
    kind = u8(queries.kind)
    pts = f64(queries.points).reshape(-1, 24)
    seps = None if per_query_min_sep is None else f64(per_query_min_sep)
    toi = _out_array(toi_out, n, np.float64, "toi_out")
    flags = _out_array(flags_out, n, np.uint8, "flags_out")
    st = abi.NarrowStats()
    ccfg = cfg.to_c()
    check(lib().ccdk_narrow_phase(c.h, p(kind, P_U8), p(pts, P_F64), p(seps, P_F64), n, C.byref(ccfg),
                                  queue_capacity, p(toi, P_F64), p(flags, P_U8), C.byref(st)))
    return NarrowOutcome(toi[:n], flags[:n], st.global_toi, bool(st.overflow),
                         int(st.peak_queue), int(st.total_splits), int(st.evaluations),
                         int(st.split_actions), int(st.generations), float(st.device_ms))


def narrow_phase_device(kind_ptr: int, points_ptr: int, n: int, cfg: NarrowConfig | None = None,
                        toi_ptr: int | None = None, flags_ptr: int | None = None,
                        sep_ptr: int | None = None, queue_capacity: int = abi.UINT64_MAX,
                        ctx=None) -> NarrowOutcome:
    """narrow_phase on device-resident queries (device pointers, e.g. from
    torch tensors); per-query results go to toi_ptr/flags_ptr when given."""
    cfg = cfg or NarrowConfig()
    c = _ctx(ctx)
    st = abi.NarrowStats()
    ccfg = cfg.to_c()
    vp = lambda x: None if x is None else C.c_void_p(int(x))
    check(lib().ccdk_narrow_phase_device(c.h, vp(kind_ptr), vp(points_ptr), vp(sep_ptr), n, C.byref(ccfg),
                                         queue_capacity, vp(toi_ptr), vp(flags_ptr), C.byref(st)))
    return NarrowOutcome(None, None, st.global_toi, bool(st.overflow), int(st.peak_queue),
                         int(st.total_splits), int(st.evaluations), int(st.split_actions),
                         int(st.generations), float(st.device_ms))


# -------------------------------------------------------------- pipeline.hpp

def _report(r: abi.Report, pairs) -> CcdReport:
    dev = {k: getattr(r, k) for k, _ in abi.Report._fields_ if k.startswith("ms_")}
    dev.update(vf_count=r.vf_count, pair_tests=r.pair_tests, total_splits=r.total_splits,
               peak_queue=r.peak_queue, evaluations=r.evaluations, split_actions=r.split_actions,
               generations=r.generations, axis=r.axis, kernel_launches=r.kernel_launches,
               sweep_slabs=r.sweep_slabs, sweep_entries=r.sweep_entries)
    return CcdReport(ToiResult(r.toi, bool(r.tolerance_hit), bool(r.zero_toi_diagnostic)),
                     int(r.candidate_count), int(r.query_count), int(r.batch_count),
                     {"CB": r.t_cb, "BP": r.t_bp, "SO/CD": r.t_socd, "NP": r.t_np},
                     int(r.tracked_peak_bytes), pairs, device=dev)


def ccd(scene: SceneStep, cfg: PipelineConfig | None = None, want_candidates: bool = True,
        ctx=None) -> CcdReport:
    """ccd (pipeline.hpp:67): the full CCD step from host buffers."""
    cfg = cfg or PipelineConfig()
    c = _ctx(ctx)
    if scene.vertices_t0.shape != scene.vertices_t1.shape:
        raise InvalidInput(abi.INVALID_INPUT, "vertex snapshots differ in length")
    r = abi.Report()
    ccfg = cfg.to_c()
    pairs = None
    with c.lock:
        check(lib().ccdk_ccd(c.h, p(scene.vertices_t0, P_F64), p(scene.vertices_t1, P_F64), scene.nv,
                             p(scene.edges, P_U32), scene.ne, p(scene.faces, P_U32), scene.nf,
                             C.byref(ccfg), C.byref(r)))
        if want_candidates:
            pairs = np.empty((r.candidate_count, 2), np.uint64)
            if r.candidate_count:
                check(lib().ccdk_fetch_pairs(c.h, p(pairs, P_U64)))
    return _report(r, pairs)


def run_batched(scene: SceneStep, boxes: Boxes, cfg: PipelineConfig, trace: BatchTrace,
                report: CcdReport | None = None, ctx=None) -> ToiResult:
    """run_batched (pipeline.hpp:78-80, pipeline.cpp:179-215) on a caller's box
    list (any order, duplicates allowed): budget-batched broad + narrow phase.
    Accumulates into `trace`; updates only the report fields the reference's
    run_batched writes (toi, counts, batch_count, BP / SO/CD / NP, the peak
    bytes as a max, candidates)."""
    c = _ctx(ctx)
    if scene.vertices_t0.shape != scene.vertices_t1.shape:
        raise InvalidInput(abi.INVALID_INPUT, "vertex snapshots differ in length")
    mn = np.ascontiguousarray(boxes.min_corner, np.float32).reshape(-1, 3)
    mx = np.ascontiguousarray(boxes.max_corner, np.float32).reshape(-1, 3)
    kd = np.ascontiguousarray(boxes.owner_kind, np.uint8)
    ix = np.ascontiguousarray(boxes.owner_index, np.uint32)
    r = abi.Report()
    ccfg = cfg.to_c()
    with c.lock:
        check(lib().ccdk_run_batched(c.h, p(scene.vertices_t0, P_F64), p(scene.vertices_t1, P_F64), scene.nv,
                                     p(scene.edges, P_U32), scene.ne, p(scene.faces, P_U32), scene.nf,
                                     p(mn, P_F32), p(mx, P_F32), p(kd, P_U8), p(ix, P_U32), len(kd),
                                     C.byref(ccfg), C.byref(r), None, None))
        pairs = None
        if report is not None:
            pairs = np.empty((r.candidate_count, 2), np.uint64)
            if r.candidate_count:
                check(lib().ccdk_fetch_pairs(c.h, p(pairs, P_U64)))
    trace.broad_batches += int(r.broad_batches)
    trace.narrow_batches += int(r.batch_count)
    toi = ToiResult(r.toi, bool(r.tolerance_hit), bool(r.zero_toi_diagnostic))
    if report is not None:
        report.toi = toi
        report.candidate_count = int(r.candidate_count)
        report.query_count = int(r.query_count)
        report.batch_count = max(1, trace.narrow_batches)
        report.per_stage_times.update({"BP": r.t_bp, "SO/CD": r.t_socd, "NP": r.t_np})
        report.tracked_peak_bytes = max(report.tracked_peak_bytes, int(r.tracked_peak_bytes))
        report.candidates = pairs
    return toi


def ccd_no_zero_toi(scene: SceneStep, cfg: PipelineConfig, want_candidates: bool = True,
                    ctx=None) -> CcdReport:
    """ccd_no_zero_toi (pipeline.hpp:82-85): the zero-ToI retry policy."""
    c = _ctx(ctx)
    r = abi.Report()
    ccfg = cfg.to_c()
    pairs = None
    with c.lock:
        check(lib().ccdk_ccd_no_zero_toi(c.h, p(scene.vertices_t0, P_F64), p(scene.vertices_t1, P_F64),
                                         scene.nv, p(scene.edges, P_U32), scene.ne, p(scene.faces, P_U32),
                                         scene.nf, C.byref(ccfg), C.byref(r)))
        if want_candidates:
            pairs = np.empty((r.candidate_count, 2), np.uint64)
            if r.candidate_count:
                check(lib().ccdk_fetch_pairs(c.h, p(pairs, P_U64)))
    return _report(r, pairs)


def query_min_separations(queries: QueryBatch, cfg: PipelineConfig, ctx=None) -> np.ndarray:
    """query_min_separations (pipeline.hpp:90-91)."""
    c = _ctx(ctx)
    n = len(queries)
    out = np.empty(max(n, 1), np.float64)
    kind, pts = u8(queries.kind), f64(queries.points).reshape(-1, 24)
    ccfg = cfg.to_c()
    check(lib().ccdk_query_min_separations(c.h, p(kind, P_U8), p(pts, P_F64), n, C.byref(ccfg),
                                           p(out, P_F64)))
    return out[:n].copy()


def point_triangle_distance(p_, a, b, c_, ctx=None) -> float:
    """distance.hpp: evaluated by the device kernel of query_min_separations
    (Relative mode with fraction 1)."""
    q = QueryBatch(np.zeros(1, np.uint8), np.concatenate([np.ravel(x) for x in (p_, a, b, c_)] + [np.zeros(12)])[None])
    return float(query_min_separations(q, PipelineConfig(min_sep_mode=MINSEP_RELATIVE, min_sep_fraction=1.0), ctx)[0])


def segment_segment_distance(p0, p1, q0, q1, ctx=None) -> float:
    q = QueryBatch(np.ones(1, np.uint8), np.concatenate([np.ravel(x) for x in (p0, p1, q0, q1)] + [np.zeros(12)])[None])
    return float(query_min_separations(q, PipelineConfig(min_sep_mode=MINSEP_RELATIVE, min_sep_fraction=1.0), ctx)[0])


class ResidentScene:
    """A scene uploaded once; ``step()`` runs the device-resident CCD step
    (the timed unit of bench.py).  ``shard`` restricts the sweep to one of
    ``shards`` equal-work slices of sorted left positions.  A context holds
    one resident scene (in its own slot: per-call uploads of ccd, build_boxes,
    classify never touch it); a second ResidentScene on the same context
    replaces the first, and the first then raises ConfigError on use, so give
    each its own Context."""

    def __init__(self, scene: SceneStep, ctx=None):
        import weakref
        self.ctx = _ctx(ctx)
        self.scene = scene
        check(lib().ccdk_scene_upload(self.ctx.h, p(scene.vertices_t0, P_F64),
                                      p(scene.vertices_t1, P_F64), scene.nv, p(scene.edges, P_U32),
                                      scene.ne, p(scene.faces, P_U32), scene.nf))
        self.ctx.resident_owner = weakref.ref(self)

    def _check_current(self):
        owner = getattr(self.ctx, "resident_owner", None)
        if owner is None or owner() is not self:
            raise ConfigError(abi.CONFIG, "ResidentScene: a later ResidentScene replaced this scene on its context")

    def step(self, cfg: PipelineConfig, shard: int = 0, shards: int = 1) -> CcdReport:
        self._check_current()
        r = abi.Report()
        ccfg = cfg.to_c()
        check(lib().ccdk_ccd_resident(self.ctx.h, C.byref(ccfg), shard, shards, C.byref(r)))
        return _report(r, None)

    def broad(self, cfg: PipelineConfig, shard: int = 0, shards: int = 1):
        """Box build + this shard's sweep + pair sort; keys stay on the device.
        Returns (n_pairs, key_bits, device_ms)."""
        self._check_current()
        n, nb, ms = C.c_uint64(), C.c_int(), C.c_float()
        ccfg = cfg.to_c()
        check(lib().ccdk_broad_resident(self.ctx.h, C.byref(ccfg), shard, shards, C.byref(n), C.byref(nb),
                                        C.byref(ms)))
        return int(n.value), int(nb.value), float(ms.value)

    def copy_keys(self, dev_ptr: int):
        """Device copy of the last broad() keys (n_pairs u64) into dev_ptr."""
        check(lib().ccdk_copy_keys_device(self.ctx.h, C.c_void_p(dev_ptr)))

    def narrow_keys(self, cfg: PipelineConfig, keys_ptr: int, n: int, key_bits: int) -> CcdReport:
        """Classify + narrow phase on n canonical pair keys in device memory."""
        self._check_current()
        r = abi.Report()
        ccfg = cfg.to_c()
        check(lib().ccdk_ccd_keys_resident(self.ctx.h, C.byref(ccfg), C.c_void_p(keys_ptr), n, key_bits,
                                           C.byref(r)))
        return _report(r, None)

    def candidates(self, n: int) -> np.ndarray:
        out = np.empty((n, 2), np.uint64)
        if n:
            check(lib().ccdk_fetch_pairs(self.ctx.h, p(out, P_U64)))
        return out

    def query_results(self, n: int):
        toi = np.empty(max(n, 1), np.float64)
        fl = np.empty(max(n, 1), np.uint8)
        if n:
            check(lib().ccdk_fetch_query_results(self.ctx.h, p(toi, P_F64), p(fl, P_U8)))
        return toi[:n], fl[:n]

    def copy_toi_to(self, dev_ptr: int):
        """Device copy of the last global ToI into ``dev_ptr`` (one double)."""
        check(lib().ccdk_copy_last_toi(self.ctx.h, C.c_void_p(dev_ptr)))

    def toi_device_ptr(self) -> int:
        v = C.c_void_p()
        check(lib().ccdk_last_toi_device_ptr(self.ctx.h, C.byref(v)))
        return int(v.value)
