"""ctypes mirror of include/ccdk.h (structs, enums, status codes)."""
from __future__ import annotations

import ctypes as C

OK, INVALID_INPUT, CONFIG, CUDA, OOM, NCCL, CAPACITY = range(7)
KIND_VERTEX, KIND_EDGE, KIND_FACE = 0, 1, 2
QUERY_VF, QUERY_EE = 0, 1
BROAD_STQ, BROAD_BF, BROAD_SAP = 0, 1, 2
MINSEP_ABSOLUTE, MINSEP_RELATIVE = 0, 1
ACTION_PRUNED, ACTION_COLLISION, ACTION_SPLIT = 0, 1, 2
FLAG_TOLERANCE_HIT, FLAG_ZERO_TOI_DIAG = 1, 2
UINT64_MAX = (1 << 64) - 1
SIZE_MAX_DIV4 = UINT64_MAX // 4


class NarrowCfg(C.Structure):
    _fields_ = [("delta", C.c_double), ("min_separation", C.c_double), ("t_max", C.c_double),
                ("max_splits", C.c_uint64), ("no_zero_toi", C.c_int32), ("reserved", C.c_int32)]


class PipelineCfg(C.Structure):
    _fields_ = [("narrow", NarrowCfg), ("broad_method", C.c_int32), ("min_sep_mode", C.c_int32),
                ("memory_budget", C.c_uint64), ("rs_params", C.c_uint64), ("rs_query", C.c_uint64),
                ("rs_interval", C.c_uint64), ("rs_pair_ints", C.c_uint64),
                ("min_sep_fraction", C.c_double), ("threads", C.c_uint32),
                ("reserved", C.c_uint32), ("inflation", C.c_double)]


class NarrowStats(C.Structure):
    _fields_ = [("global_toi", C.c_double), ("overflow", C.c_int32), ("reserved", C.c_int32),
                ("peak_queue", C.c_uint64), ("total_splits", C.c_uint64),
                ("evaluations", C.c_uint64), ("split_actions", C.c_uint64),
                ("generations", C.c_uint64), ("device_ms", C.c_double)]


class StqStats(C.Structure):
    _fields_ = [("max_queue", C.c_uint64), ("n_rounds", C.c_uint64),
                ("pair_tests", C.c_uint64), ("axis", C.c_uint64),
                ("axis_flags", C.c_uint64)]


class Report(C.Structure):
    _fields_ = [("toi", C.c_double), ("tolerance_hit", C.c_uint8),
                ("zero_toi_diagnostic", C.c_uint8), ("reserved", C.c_uint8 * 6),
                ("candidate_count", C.c_uint64), ("query_count", C.c_uint64),
                ("batch_count", C.c_uint64), ("t_cb", C.c_double), ("t_bp", C.c_double),
                ("t_socd", C.c_double), ("t_np", C.c_double),
                ("tracked_peak_bytes", C.c_uint64), ("vf_count", C.c_uint64),
                ("pair_tests", C.c_uint64), ("total_splits", C.c_uint64),
                ("peak_queue", C.c_uint64), ("evaluations", C.c_uint64),
                ("split_actions", C.c_uint64), ("generations", C.c_uint64),
                ("axis", C.c_int32), ("reserved2", C.c_int32),
                ("ms_build", C.c_double), ("ms_sort", C.c_double), ("ms_sweep", C.c_double),
                ("ms_pairsort", C.c_double), ("ms_classify", C.c_double),
                ("ms_narrow", C.c_double), ("ms_total", C.c_double),
                ("kernel_launches", C.c_uint64), ("broad_batches", C.c_uint64),
                ("sweep_slabs", C.c_uint64), ("sweep_entries", C.c_uint64)]


def narrow_cfg(delta=1e-6, min_separation=0.0, t_max=1.0, max_splits=1 << 20,
               no_zero_toi=False) -> NarrowCfg:
    """NarrowConfig defaults (narrowphase.hpp:31-39)."""
    return NarrowCfg(delta, min_separation, t_max, max_splits, int(bool(no_zero_toi)), 0)


def pipeline_cfg(narrow: NarrowCfg | None = None, broad_method=BROAD_STQ,
                 memory_budget=SIZE_MAX_DIV4, min_sep_mode=MINSEP_ABSOLUTE,
                 min_sep_fraction=0.2, threads=1, inflation=0.0,
                 record_sizes=(56, 192, 252, 8)) -> PipelineCfg:
    """PipelineConfig defaults (pipeline.hpp:34-45); inflation defaults to
    0.0 there, the BASELINE configs set 0.01 explicitly."""
    p = PipelineCfg()
    p.narrow = narrow if narrow is not None else narrow_cfg()
    p.broad_method = broad_method
    p.min_sep_mode = min_sep_mode
    p.memory_budget = memory_budget
    p.rs_params, p.rs_query, p.rs_interval, p.rs_pair_ints = record_sizes
    p.min_sep_fraction = min_sep_fraction
    p.threads = threads
    p.inflation = inflation
    return p


def ptr(a, ctype):
    """Pointer to a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


P_F64 = C.POINTER(C.c_double)
P_F32 = C.POINTER(C.c_float)
P_U8 = C.POINTER(C.c_uint8)
P_U16 = C.POINTER(C.c_uint16)
P_U32 = C.POINTER(C.c_uint32)
P_U64 = C.POINTER(C.c_uint64)
