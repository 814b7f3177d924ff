/*
 * ccdk.h — the C ABI of the B200-native conservative CCD hot path.
 *
 * This is the drop-in boundary.  The reference (ccdkit, a CPU-only C++20
 * library) has no FFI: its boundary is the C++ header API under
 * proj/include/ccdkit/*.hpp, replaced at link time.  Every entry point below
 * is the plain-pointer restatement of one of those C++ functions; the C++
 * shim in paper_2112_06300_b200/csrc/ccdkit_host.cpp re-exposes them with
 * the reference signatures (include/ccdkit/*.hpp), and the Python package
 * binds them with ctypes.
 *
 * Conventions (mirroring the reference's error behaviour):
 *   - every function returns a ccdk_status; CCDK_INVALID_INPUT maps to
 *     ccdkit::InvalidInput and CCDK_CONFIG to ccdkit::ConfigError;
 *     ccdk_last_error() returns the thread-local message of the last failure;
 *   - calls on one context are serialised by its mutex; results a context
 *     holds for a later fetch (candidate pairs, round sizes, per-query
 *     results, the resident scene) belong to its last producing call, so a
 *     caller sharing a context across threads holds its own lock around a
 *     produce-then-fetch sequence (the C++ shim and the Python package do);
 *   - all array arguments are HOST pointers unless the name ends in _dev;
 *   - a primitive id is packed as (kind << 32) | index (kind 0 = vertex,
 *     1 = edge, 2 = face), so u64 order equals the reference's PrimitiveId
 *     order (scene.hpp:13-26); a candidate pair is two such ids, left < right;
 *   - a narrow query is 24 doubles: points_t0[4][3] then points_t1[4][3]
 *     (NarrowQuery, broadphase.hpp:26-35), plus a kind byte (0 = VF, 1 = EE).
 *
 * There is no CPU fallback: if no CUDA device is usable every compute entry
 * point fails with CCDK_CUDA.
 */
#ifndef CCDK_H
#define CCDK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CCDK_ABI_VERSION 2 /* 2: ccdk_report gained sweep_slabs, sweep_entries; ccdk_ccd_into,
                              ccdk_run_batched */

#if defined(__GNUC__)
#define CCDK_API __attribute__((visibility("default")))
#else
#define CCDK_API
#endif

typedef enum {
    CCDK_OK = 0,
    CCDK_INVALID_INPUT = 1, /* ccdkit::InvalidInput (core.hpp:47-53) */
    CCDK_CONFIG = 2,        /* ccdkit::ConfigError  (core.hpp:55-61) */
    CCDK_CUDA = 3,          /* CUDA runtime failure or no device */
    CCDK_OOM = 4,           /* device allocation failed */
    CCDK_NCCL = 5,          /* collective failure (multi-GPU host layer) */
    CCDK_CAPACITY = 6       /* device work buffer full: caller halves the batch */
} ccdk_status;

enum { CCDK_KIND_VERTEX = 0, CCDK_KIND_EDGE = 1, CCDK_KIND_FACE = 2 };
enum { CCDK_QUERY_VF = 0, CCDK_QUERY_EE = 1 };
enum { CCDK_BROAD_STQ = 0, CCDK_BROAD_BF = 1, CCDK_BROAD_SAP = 2 };
enum { CCDK_MINSEP_ABSOLUTE = 0, CCDK_MINSEP_RELATIVE = 1 };
enum { CCDK_ACTION_PRUNED = 0, CCDK_ACTION_COLLISION = 1, CCDK_ACTION_SPLIT = 2 };

#define CCDK_FLAG_TOLERANCE_HIT 1u
#define CCDK_FLAG_ZERO_TOI_DIAG 2u

/* NarrowConfig (narrowphase.hpp:31-39). */
typedef struct {
    double delta;          /* 1e-6 */
    double min_separation; /* 0    */
    double t_max;          /* 1    */
    uint64_t max_splits;   /* 2^20 */
    int32_t no_zero_toi;   /* 0    */
    int32_t reserved;
} ccdk_narrow_cfg;

/* PipelineConfig (pipeline.hpp:34-45) incl. RecordSizes (pipeline.hpp:22-27). */
typedef struct {
    ccdk_narrow_cfg narrow;
    int32_t broad_method;    /* CCDK_BROAD_* */
    int32_t min_sep_mode;    /* CCDK_MINSEP_* */
    uint64_t memory_budget;  /* SIZE_MAX/4 = unbounded */
    uint64_t rs_params;      /* 56  */
    uint64_t rs_query;       /* 192 */
    uint64_t rs_interval;    /* 252 */
    uint64_t rs_pair_ints;   /* 8   */
    double min_sep_fraction; /* 0.2 */
    uint32_t threads;        /* accepted and ignored (advisory in the reference) */
    uint32_t reserved;
    double inflation;        /* 0.0 */
} ccdk_pipeline_cfg;

/* NarrowOutcome scalars (narrowphase.hpp:84-90) plus device work counters. */
typedef struct {
    double global_toi;
    int32_t overflow;
    int32_t reserved;
    uint64_t peak_queue;
    uint64_t total_splits;
    uint64_t evaluations;    /* evaluate_box calls (roofline E) */
    uint64_t split_actions;  /* Split actions incl. budget-rejected (roofline S) */
    uint64_t generations;    /* BFS generations executed */
    double device_ms;        /* CUDA-event time of the narrow phase */
} ccdk_narrow_stats;

/* StqStats (broadphase.hpp:45-48) plus sweep work counters. */
typedef struct {
    uint64_t max_queue;
    uint64_t n_rounds;       /* length of round_sizes; fetch with ccdk_fetch_round_sizes */
    uint64_t pair_tests;     /* sum of run lengths over the left range (roofline T) */
    uint64_t axis;
    uint64_t axis_flags;     /* bit0: tree variances within the error bound of a tie,
                                bit1: axis decided by the reference's serial sums */
} ccdk_stq_stats;

/* CcdReport (pipeline.hpp:47-61); stage times in seconds like the reference. */
typedef struct {
    double toi;
    uint8_t tolerance_hit;
    uint8_t zero_toi_diagnostic;
    uint8_t reserved[6];
    uint64_t candidate_count;
    uint64_t query_count;
    uint64_t batch_count;
    double t_cb, t_bp, t_socd, t_np; /* "CB", "BP", "SO/CD", "NP" */
    uint64_t tracked_peak_bytes;
    /* device detail (not in the reference report) */
    uint64_t vf_count;
    uint64_t pair_tests;
    uint64_t total_splits;
    uint64_t peak_queue;
    uint64_t evaluations;
    uint64_t split_actions;
    uint64_t generations;
    int32_t axis;
    int32_t reserved2;
    double ms_build, ms_sort, ms_sweep, ms_pairsort, ms_classify, ms_narrow, ms_total;
    uint64_t kernel_launches; /* own (non-CUB) kernels launched by this step */
    uint64_t broad_batches;   /* BatchTrace::broad_batches */
    uint64_t sweep_slabs;     /* slab-mode sweep: slab count (0 = 1-D sweep) */
    uint64_t sweep_entries;   /* slab-mode sweep: boxes incl. their copies in further slabs */
} ccdk_report;

typedef struct ccdk_ctx ccdk_ctx;

/* ---- context ------------------------------------------------------------ */
CCDK_API int ccdk_abi_version(void);
CCDK_API const char* ccdk_last_error(void);
CCDK_API int ccdk_ctx_create(int device, ccdk_ctx** out);
CCDK_API int ccdk_ctx_destroy(ccdk_ctx* ctx);
/* Run all work of this context on `stream` (a cudaStream_t); NULL = a private
 * non-blocking stream of the context (the default: NOT ordered with any other
 * stream).  To share the legacy default stream pass cudaStreamLegacy (0x1). */
CCDK_API int ccdk_ctx_set_stream(ccdk_ctx* ctx, void* stream);
CCDK_API int ccdk_ctx_synchronize(ccdk_ctx* ctx);
/* Narrow-phase interval buffer capacity (intervals per generation buffer).
 * 0 = size from free device memory. Exceeding it returns CCDK_CAPACITY. */
CCDK_API int ccdk_ctx_set_interval_capacity(ccdk_ctx* ctx, uint64_t intervals);

/* ---- geometry: aabb.hpp ------------------------------------------------- */
/* round_down_reduced / round_up_reduced (aabb.hpp:10-14, aabb.cpp:10-28),
 * batched; non-finite input -> CCDK_INVALID_INPUT. */
CCDK_API int ccdk_round_reduced(ccdk_ctx* ctx, const double* x, uint64_t n, float* down, float* up);

/* build_boxes (aabb.hpp:49-50, aabb.cpp:71-112).  Scene layout: vertices as
 * nv*3 doubles per snapshot, edges ne*2 u32, faces nf*3 u32.  Outputs k =
 * nv+ne+nf boxes: min/max k*3 floats, owner kind (u8) and index (u32). */
CCDK_API int ccdk_build_boxes(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                     const uint32_t* edges, uint64_t ne, const uint32_t* faces,
                     uint64_t nf, double inflation, float* min_corner,
                     float* max_corner, uint8_t* owner_kind, uint32_t* owner_index);

/* ---- broad phase: broadphase.hpp ---------------------------------------- */
/* choose_axis (broadphase.hpp:51, broadphase.cpp:45-67). */
CCDK_API int ccdk_choose_axis(ccdk_ctx* ctx, const float* min_corner, const float* max_corner,
                     uint64_t k, int* axis);

/* stq / bf / sap (broadphase.hpp:57-68) over arbitrary boxes.  Result pairs
 * stay on the device in ctx; *n_pairs receives the count, fetch them with
 * ccdk_fetch_pairs.  range_end = UINT64_MAX means unrestricted. */
CCDK_API int ccdk_broad_phase(ccdk_ctx* ctx, int method, const float* min_corner,
                     const float* max_corner, const uint8_t* owner_kind,
                     const uint32_t* owner_index, uint64_t k, uint64_t nv,
                     const uint32_t* edges, uint64_t ne, const uint32_t* faces,
                     uint64_t nf, uint64_t range_begin, uint64_t range_end,
                     uint64_t* n_pairs, ccdk_stq_stats* stats);
/* Copy the last pair list: out holds 2*n_pairs u64 (left id, right id). */
CCDK_API int ccdk_fetch_pairs(ccdk_ctx* ctx, uint64_t* out);
/* Copy StqStats::round_sizes of the last broad phase (n_rounds entries). */
CCDK_API int ccdk_fetch_round_sizes(ccdk_ctx* ctx, uint64_t* out);

/* classify (broadphase.hpp:78-79, broadphase.cpp:194-239): pairs (2*n u64)
 * -> VF queries then EE queries (pipeline.cpp:162-165 order).  Output
 * arrays must hold n entries; *n_vf and *n_ee receive the counts. */
CCDK_API int ccdk_classify(ccdk_ctx* ctx, const uint64_t* pairs, uint64_t n_pairs,
                  const double* v0, const double* v1, uint64_t nv,
                  const uint32_t* edges, uint64_t ne, const uint32_t* faces,
                  uint64_t nf, uint8_t* kind_out, double* points_out,
                  uint64_t* source_out, uint64_t* n_vf, uint64_t* n_ee);

/* ---- narrow phase: narrowphase.hpp ------------------------------------- */
/* inclusion_box (narrowphase.hpp:59) batched: box = (tlo,thi,ulo,uhi,vlo,vhi)
 * per entry; out = 6 doubles (x.lo,x.hi,y.lo,y.hi,z.lo,z.hi). */
CCDK_API int ccdk_inclusion_boxes(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                         const double* boxes, uint64_t n, double* out);

/* process_interval (narrowphase.hpp:77-79) batched.  depth = 3 u16 per box;
 * sep < 0 means cfg.min_separation.  action[i] in CCDK_ACTION_*; for Split,
 * children = 12 doubles (left box, right box) and child_depth = 6 u16. */
CCDK_API int ccdk_process_intervals(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                           const double* boxes, const uint16_t* depth,
                           const double* t_star, const double* sep, uint64_t n,
                           const ccdk_narrow_cfg* cfg, uint8_t* action,
                           double* candidate_t, uint8_t* zero_diag, double* children,
                           uint16_t* child_depth);

/* narrow_phase (narrowphase.hpp:97-100, narrowphase.cpp:189-311).
 * per_query_sep may be NULL.  toi/flags hold n entries (flags bit0 =
 * tolerance_hit, bit1 = zero_toi_diagnostic).  queue_capacity = UINT64_MAX
 * for unbounded.  On semantic overflow stats->overflow = 1 and per-query
 * results are the defaults, as in the reference. */
CCDK_API int ccdk_narrow_phase(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                      const double* per_query_sep, uint64_t n,
                      const ccdk_narrow_cfg* cfg, uint64_t queue_capacity,
                      double* toi, uint8_t* flags, ccdk_narrow_stats* stats);

/* narrow_phase on device-resident queries: kind/points/per_query_sep/toi/
 * flags are DEVICE pointers (toi/flags may be NULL: results then stay in the
 * context).  Same semantics and stats as ccdk_narrow_phase; used for the
 * device-timed narrow-only benchmark (BASELINE config 5) and by multi-GPU
 * hosts that shard queries on the device. */
CCDK_API int ccdk_narrow_phase_device(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                                      const double* per_query_sep, uint64_t n,
                                      const ccdk_narrow_cfg* cfg, uint64_t queue_capacity,
                                      double* toi, uint8_t* flags, ccdk_narrow_stats* stats);

/* ---- pipeline: pipeline.hpp --------------------------------------------- */
/* ccd (pipeline.hpp:67, pipeline.cpp:218-232): the full CCD step from host
 * buffers (H2D copy, box build, broad phase, classify, narrow phase, global
 * min, D2H of the report).  Candidates stay on the device: fetch with
 * ccdk_fetch_pairs (report->candidate_count pairs, canonical order). */
CCDK_API int ccdk_ccd(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
             const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf,
             const ccdk_pipeline_cfg* cfg, ccdk_report* report);

/* Candidate export for ccdk_ccd_into.  Called twice per step: first with
 * pairs == NULL and the final candidate count (the caller may allocate and
 * fault in its destination while the list is still being copied), then with
 * the final canonical candidate list in pinned host memory that is valid only
 * during the call: 16 bytes per pair, left id then right id, each id
 * {uint8 kind, 3 zero bytes, uint32 index} (= kind | index << 32 as a
 * little-endian u64, the in-memory layout of ccdkit::CandidatePair on
 * x86-64).  When the step needs a single broad batch (always at the default
 * memory budget) the sink runs on a library worker thread WHILE the device
 * runs classify + narrow phase, so a caller's allocation and copy of the
 * list overlap the GPU; otherwise it runs on the calling thread before
 * ccdk_ccd_into returns.  Return 0, or nonzero to fail the call with
 * CCDK_OOM (e.g. the caller could not allocate; no second call follows). */
typedef int (*ccdk_pairs_sink)(void* user, const uint64_t* pairs, uint64_t n_pairs);

/* ccd returning the candidate list through `sink` (the drop-in's
 * ccdkit::ccd: CcdReport::candidates, pipeline.cpp:209). */
CCDK_API int ccdk_ccd_into(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                           const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf,
                           const ccdk_pipeline_cfg* cfg, ccdk_report* report, ccdk_pairs_sink sink,
                           void* user);

/* run_batched (pipeline.hpp:78-80, pipeline.cpp:179-215) on a caller's box
 * list: k boxes as min_corner/max_corner [k][3] floats and owners (kind,
 * index), any order, duplicates allowed.  No box build (cfg->inflation is
 * not used); broad batches halve sorted positions for stq/sap and raw box
 * positions for bf, as the reference does.  Every owner must name an
 * existing primitive (CCDK_INVALID_INPUT otherwise; the reference would
 * index out of bounds).  The scene is validated like ccdk_ccd's.  Candidates
 * go to `sink` as in ccdk_ccd_into (sink may be NULL: they stay in the
 * context for ccdk_fetch_pairs); report->broad_batches and
 * report->batch_count are BatchTrace's broad_batches and narrow_batches. */
CCDK_API int ccdk_run_batched(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                              const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf,
                              const float* min_corner, const float* max_corner, const uint8_t* owner_kind,
                              const uint32_t* owner_index, uint64_t k, const ccdk_pipeline_cfg* cfg,
                              ccdk_report* report, ccdk_pairs_sink sink, void* user);

/* ccd_no_zero_toi (pipeline.hpp:82-85, pipeline.cpp:234-256): requires
 * cfg->narrow.no_zero_toi; a separated run, then on an exact-zero ToI a
 * zero-separation always-split-at-t=0 retry whose ToI is scaled by 0.8. */
CCDK_API int ccdk_ccd_no_zero_toi(ccdk_ctx* ctx, const double* v0, const double* v1,
                                  uint64_t nv, const uint32_t* edges, uint64_t ne,
                                  const uint32_t* faces, uint64_t nf,
                                  const ccdk_pipeline_cfg* cfg, ccdk_report* report);

/* query_min_separations (pipeline.hpp:90-91, pipeline.cpp:39-55): Absolute
 * mode copies cfg->narrow.min_separation; Relative mode is min_sep_fraction
 * times the t=0 point-triangle / segment-segment distance (distance.cpp). */
CCDK_API int ccdk_query_min_separations(ccdk_ctx* ctx, const uint8_t* kind,
                                        const double* points, uint64_t n,
                                        const ccdk_pipeline_cfg* cfg, double* out);

/* Device-resident variant: upload a scene once, then run steps on it. */
CCDK_API int ccdk_scene_upload(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                      const uint32_t* edges, uint64_t ne, const uint32_t* faces,
                      uint64_t nf);
/* Full step on the uploaded scene.  shard_count > 1 restricts the sweep to
 * this shard's slice of sorted left positions (equal pair-test work per
 * shard, SweepRange semantics of broadphase.hpp:37-43); the caller combines
 * shards with an allreduce(min) of report->toi. */
CCDK_API int ccdk_ccd_resident(ccdk_ctx* ctx, const ccdk_pipeline_cfg* cfg, uint32_t shard_rank,
                      uint32_t shard_count, ccdk_report* report);
/* Multi-GPU rebalance: the step split at the candidate list.
 * ccdk_broad_resident runs the box build and this shard's STQ sweep + pair
 * sort on the uploaded scene; the shard's canonical pair keys
 * (lo_rank << key_bits | hi_rank, u64) stay on the device; copy them out with
 * ccdk_copy_keys_device (n_pairs * 8 bytes).  ccdk_ccd_keys_resident then
 * classifies and narrow-phases ANY slice of such keys (device memory, any
 * order; sorted internally): per-query results are partition-independent
 * (narrowphase.hpp:93-96), so ranks can exchange keys to equalise counts. */
CCDK_API int ccdk_broad_resident(ccdk_ctx* ctx, const ccdk_pipeline_cfg* cfg, uint32_t shard_rank,
                                 uint32_t shard_count, uint64_t* n_pairs, int* key_bits,
                                 float* device_ms);
CCDK_API int ccdk_copy_keys_device(ccdk_ctx* ctx, void* dst_dev);
CCDK_API int ccdk_ccd_keys_resident(ccdk_ctx* ctx, const ccdk_pipeline_cfg* cfg,
                                    const uint64_t* dev_keys, uint64_t n, int key_bits,
                                    ccdk_report* report);

/* Device pointer (double) holding the last step's global ToI, for a
 * device-side allreduce(min) by the multi-GPU host layer. */
CCDK_API int ccdk_last_toi_device_ptr(ccdk_ctx* ctx, void** dev_ptr);

/* Copy the last step's global ToI (one double) to device memory `dst_dev`
 * on the context stream (feeds a device-side allreduce(min)). */
CCDK_API int ccdk_copy_last_toi(ccdk_ctx* ctx, void* dst_dev);

/* Per-query results of the last ccd step (query_count entries). */
CCDK_API int ccdk_fetch_query_results(ccdk_ctx* ctx, double* toi, uint8_t* flags);

#ifdef __cplusplus
}
#endif

#endif /* CCDK_H */
