// Internal declarations shared by the ccdk translation units.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <future>
#include <string>
#include <thread>
#include <vector>

#include "ccdk.h"

namespace ccdk {

// ------------------------------------------------------------------ errors

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define CCDK_CUDA_CHECK(expr)                                                          \
    do {                                                                               \
        cudaError_t err__ = (expr);                                                    \
        if (err__ != cudaSuccess) {                                                    \
            if (err__ == cudaErrorMemoryAllocation)                                    \
                throw ::ccdk::Error(CCDK_OOM, std::string(#expr) + ": "                \
                                                  + cudaGetErrorString(err__));        \
            throw ::ccdk::Error(CCDK_CUDA, std::string(__FILE__) + ":"                 \
                                               + std::to_string(__LINE__) + " " #expr  \
                                               ": " + cudaGetErrorString(err__));      \
        }                                                                              \
    } while (0)

#define CCDK_LAUNCH_CHECK()                                                             \
    do {                                                                                \
        CCDK_CUDA_CHECK(cudaGetLastError());                                            \
        if (::ccdk::debug_enabled()) {                                                  \
            cudaError_t e__ = cudaDeviceSynchronize();                                  \
            std::fprintf(stderr, "[ccdk] %s:%d %s\n", __FILE__, __LINE__,               \
                         cudaGetErrorString(e__));                                      \
            CCDK_CUDA_CHECK(e__);                                                       \
        }                                                                               \
    } while (0)

inline bool debug_enabled()
{
    static const bool d = std::getenv("CCDK_DEBUG") != nullptr;
    return d;
}

// Debug tracing (CCDK_DEBUG=1): synchronise and report each stage.
#define CCDK_TRACE(c, msg)                                                              \
    do {                                                                                \
        if (::ccdk::debug_enabled()) {                                                  \
            cudaError_t e__ = cudaStreamSynchronize((c).stream);                        \
            std::fprintf(stderr, "[ccdk] %s: %s\n", msg, cudaGetErrorString(e__));      \
        }                                                                               \
    } while (0)

// ------------------------------------------------------------ device memory

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release()
    {
        if (p)
            cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    // grow-only; contents are not preserved
    void* ensure(size_t bytes)
    {
        if (bytes == 0)
            bytes = 16;
        if (bytes > cap) {
            release();
            size_t c = bytes + bytes / 4;
            CCDK_CUDA_CHECK(cudaMalloc(&p, c));
            cap = c;
        }
        return p;
    }
    // grow-only, preserving the first `cap` bytes (stream-ordered copy)
    void* ensure_keep(size_t bytes, cudaStream_t s)
    {
        if (bytes > cap) {
            void* np = nullptr;
            const size_t c = bytes + bytes / 2;
            CCDK_CUDA_CHECK(cudaMalloc(&np, c));
            if (p) {
                CCDK_CUDA_CHECK(cudaMemcpyAsync(np, p, cap, cudaMemcpyDeviceToDevice, s));
                CCDK_CUDA_CHECK(cudaStreamSynchronize(s));
                cudaFree(p);
            }
            p = np;
            cap = c;
        }
        return p;
    }
    template <typename T>
    T* as() const
    {
        return static_cast<T*>(p);
    }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~PinnedBuf()
    {
        if (p)
            cudaFreeHost(p);
    }
    void* ensure(size_t bytes)
    {
        if (bytes > cap) {
            if (p)
                cudaFreeHost(p);
            p = nullptr;
            CCDK_CUDA_CHECK(cudaMallocHost(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    template <typename T>
    T* as() const
    {
        return static_cast<T*>(p);
    }
};

// Timing events, created once per context (creating/destroying events per
// call takes driver locks; fixed slots per call site, each slot's use is
// synchronised before its next record).
struct EventPool {
    enum { kStep = 0, kBatch = 6, kBroad = 8, kNarrow = 12, kApi = 16, kExport = 20, kSlots = 22 };
    cudaEvent_t ev[kSlots] = {};
    EventPool() = default;
    EventPool(const EventPool&) = delete;
    EventPool& operator=(const EventPool&) = delete;
    ~EventPool()
    {
        for (auto e : ev)
            if (e)
                cudaEventDestroy(e);
    }
    cudaEvent_t get(int i)
    {
        if (!ev[i]) {
            const cudaError_t r = cudaEventCreate(&ev[i]);
            if (r != cudaSuccess)
                throw Error(CCDK_CUDA, std::string("cudaEventCreate: ") + cudaGetErrorString(r));
        }
        return ev[i];
    }
};

// Persistent host helper threads of a context (staging copies of pageable
// uploads): spawning threads per call cost more than the copies they share.
// run(f, k) runs f on k helpers and the caller and returns when all are done.
class HostPool {
public:
    HostPool() = default;
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;
    ~HostPool()
    {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_)
            t.join();
    }
    template <class F>
    void run(F&& f, unsigned helpers)
    {
        start(std::forward<F>(f), helpers);
        (*task_)();
        wait();
    }
    // run f on `helpers` threads and return at once; wait() joins them
    template <class F>
    void start(F&& f, unsigned helpers)
    {
        ensure(helpers);
        {
            std::lock_guard<std::mutex> lk(m_);
            task_store_ = std::function<void()>(std::forward<F>(f));
            task_ = &task_store_;
            want_ = helpers;
            busy_ = helpers;
            ++gen_;
        }
        cv_.notify_all();
    }
    void wait()
    {
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return busy_ == 0; });
        task_ = nullptr;
    }

private:
    void ensure(unsigned n)
    {
        while (threads_.size() < n) {
            const unsigned id = static_cast<unsigned>(threads_.size());
            threads_.emplace_back([this, id] { loop(id); });
        }
    }
    void loop(unsigned id)
    {
        unsigned long long seen = 0;
        for (;;) {
            std::function<void()>* t;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && id < want_); });
                if (stop_)
                    return;
                seen = gen_;
                t = task_;
            }
            (*t)();
            {
                std::lock_guard<std::mutex> lk(m_);
                --busy_;
            }
            done_.notify_one();
        }
    }
    std::vector<std::thread> threads_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::function<void()>* task_ = nullptr;
    std::function<void()> task_store_;
    unsigned want_ = 0, busy_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

// Device-side scene (canonical slot order V, E, F; aabb.cpp:79-105).
struct DevScene {
    DevBuf v0, v1, edges, faces;
    uint64_t nv = 0, ne = 0, nf = 0;
    bool valid = false;
};

// Device work counters, one struct in device memory per context.
struct DevCounters {
    unsigned long long n_pairs;       // sweep output cursor
    unsigned long long pair_tests;    // sum of run lengths in the range
    unsigned long long n_heavy;       // heavy sweep segments
    unsigned long long error;         // first error code seen by a kernel
    unsigned long long misc[4];
};

// Narrow-phase device scalars.
struct NarrowScalars {
    unsigned long long cur_n;       // intervals in the current generation
    unsigned long long next_n;      // append cursor of the next generation
    unsigned long long dirty_n;     // queries whose ToI dropped this generation
    unsigned long long dropped;     // intervals of exhausted queries dropped
    unsigned long long evaluations;
    unsigned long long split_actions;
    unsigned long long peak;        // max compacted queue size
    unsigned long long gen;         // generation index
    unsigned long long cont;        // 1 while another generation is needed
    unsigned long long sem_overflow;
    unsigned long long phys_overflow;
    unsigned long long finish_ticket;
    unsigned long long total_splits;
    unsigned long long global_toi_bits;
    unsigned long long any_flags;   // OR of per-query flags
    unsigned long long vf_count;
    unsigned long long gen_limit;   // set when the generation guard trips
    unsigned long long nq;            // queries of this run (device-side so the graph is size-independent)
    unsigned long long dirty_cap;     // dirty-list capacity; beyond it every query is refreshed
    unsigned long long cur_pairs[3];  // split records per region in the current generation
    unsigned long long next_pairs[3]; // append cursors of the next generation
    unsigned long long exh_next;      // next-generation intervals of exhausted queries (exact-size scans)
    unsigned long long stopped;       // the run stopped at GenArgs::gen_stop
};

// The narrow phase's generation loop as one CUDA graph: a WHILE conditional
// node whose body is k_generation -> k_finish; k_finish clears the condition
// when no further generation is needed, so the whole BFS runs without a host
// round trip.  Re-instantiated only when the kernel arguments change.
struct GenGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    unsigned char key[1024];
    size_t key_size = 0;
    GenGraph() = default;
    GenGraph(const GenGraph&) = delete;
    GenGraph& operator=(const GenGraph&) = delete;
    ~GenGraph() { reset(); }
    void reset()
    {
        if (exec)
            cudaGraphExecDestroy(exec);
        if (graph)
            cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        key_size = 0;
    }
};

struct Ctx;

// -------------------------------------------------------- kernel launchers
// geometry (ccdk_geometry.cu)
void launch_round(Ctx& c, const double* x, uint64_t n, float* dn, float* up);
// build canonical boxes: SoA mins/maxs [3][k], owner vertex triples + rank.
void launch_build_boxes(Ctx& c, const double* v0, const double* v1, uint64_t nv,
                        const uint32_t* e, uint64_t ne, const uint32_t* f, uint64_t nf,
                        double inflation, float* bmin, float* bmax, uint4* vids);
void launch_soa_to_aos(Ctx& c, const float* bmin, const float* bmax, uint64_t k, float* mn,
                       float* mx, uint8_t* kind, uint32_t* index, uint64_t nv, uint64_t ne);

// broad phase (ccdk_broad.cu)
struct BroadOut {
    uint64_t n_pairs = 0;     // candidates (canonical, unique)
    uint64_t pair_tests = 0;
    uint64_t range_lo = 0, range_hi = 0; // sorted left positions actually swept
    int axis = 0;
    bool axis_near_tie = false; // tree-summed variances within the error bound of a tie
    bool axis_serial = false;   // ... and the reference's serial order decided the axis
    float ms_axis_sort = 0, ms_sweep = 0, ms_pairsort = 0;
    bool slab_mode = false;     // the sweep ran per slab (K5'); entries = boxes incl. slab copies
    uint64_t launches = 0;      // own (non-CUB) kernels launched
    uint64_t slab_count = 0, slab_entries = 0;
};
// General broad phase over SoA boxes whose slot order is owner order (rank =
// slot) or, with owner arrays, an arbitrary box list.
struct BroadIn {
    const float* bmin = nullptr; // [3][k]
    const float* bmax = nullptr;
    const uint4* vids = nullptr; // (v0, v1, v2, rank); absent vertices = 0xffffffff
    const uint32_t* raw = nullptr; // raw input position per slot (bf ranges); null = identity
    uint64_t k = 0;
    int method = CCDK_BROAD_STQ;
    uint64_t range_begin = 0, range_end = UINT64_MAX;
    uint32_t shard_rank = 0, shard_count = 1;
    bool want_rounds = false;
    bool unique = false; // duplicate owners possible
    int rank_bits = 0;   // bits of the vids' rank space; 0 = ceil_log2(k)
    // reproduce choose_axis's serial summation order on near ties (the axis
    // is observable through choose_axis, StqStats and SweepRange slices)
    bool exact_axis = true;
    bool allow_slab = true; // slab-mode sweep permitted (full range, no StqStats)
    // the box build's non-finite flag (DevCounters::error) is checked at the
    // broad phase's first read-back instead of its own host round trip
    bool check_build_error = false;
    // leave the stage times / axis for broad_collect() (the caller syncs later)
    bool defer_collect = false;
};
void broad_collect(Ctx& c, BroadOut& out);
void broad_phase(Ctx& c, const BroadIn& in, BroadOut& out);

// narrow phase (ccdk_narrow.cu)
// Fused K7 + generation 0: the candidate keys and the scene a narrow run
// classifies from itself (k_classify_gen0 writes the query records while it
// evaluates the roots from registers).  Set in Ctx::classify_pending by the
// pipeline; any path that cannot fuse calls ensure_classified() first.
struct ClassifySrc {
    const uint64_t* keys = nullptr;
    uint64_t n = 0;
    int nb = 0;
    const double* v0 = nullptr;
    const double* v1 = nullptr;
    uint64_t nv = 0;
    const uint32_t* e = nullptr;
    uint64_t ne = 0;
    const uint32_t* f = nullptr;
    uint8_t* kind_out = nullptr;
    double* pts_out = nullptr;
    uint32_t* qflags_out = nullptr;
};
void ensure_classified(Ctx& c);

struct NarrowIn {
    const uint8_t* kind = nullptr;   // device
    const double* points = nullptr;  // device, n*24, internal order (iv::GlobalPtsIL)
    const double* sep = nullptr;     // device or null
    const uint32_t* qflags = nullptr; // device or null: per-query kind | exact-widening flags precomputed
    uint64_t n = 0;
    ccdk_narrow_cfg cfg {};
    uint64_t queue_capacity = UINT64_MAX;
};
struct NarrowOut {
    ccdk_narrow_stats stats {};
    double* toi = nullptr;     // device, n (owned by ctx)
    uint8_t* flags = nullptr;  // device, n
    uint64_t launches = 0;     // generation + finish kernels launched
    uint64_t any_flags = 0;    // OR of the per-query flags
};
void narrow_phase(Ctx& c, const NarrowIn& in, NarrowOut& out);
void launch_inclusion(Ctx& c, const uint8_t* kind, const double* pts, const double* boxes,
                      uint64_t n, double* out);
void launch_process(Ctx& c, const uint8_t* kind, const double* pts, const double* boxes,
                    const uint16_t* depth, const double* t_star, const double* sep, uint64_t n,
                    const ccdk_narrow_cfg& cfg, uint8_t* action, double* cand_t,
                    uint8_t* zdiag, double* children, uint16_t* child_depth);
// classify canonical keys (lo<<nb | hi, ranks = slots) into queries
void launch_classify_keys(Ctx& c, const uint64_t* keys, uint64_t n, int nb,
                          const double* v0, const double* v1, uint64_t nv,
                          const uint32_t* e, uint64_t ne, const uint32_t* f, uint8_t* kind,
                          double* pts, uint32_t* qflags);
// query_min_separations (pipeline.cpp:39-55) incl. the distances of
// distance.cpp (ccdk_distance.cu); internal: records in internal order
void launch_min_seps(Ctx& c, const uint8_t* kind, const double* pts, uint64_t n,
                     const ccdk_pipeline_cfg& cfg, double* out, bool internal);
// device-to-device copy by a kernel (stays off the copy engines)
void launch_copy_device(Ctx& c, const void* src, void* dst, uint64_t bytes);
// reference-order query records -> narrow-phase internal order
void launch_records_to_internal(Ctx& c, const double* ref, uint64_t n, double* il);
// layout 0: (kind << 32) | index per id (C ABI); layout 1: kind | index << 32
// (ccdkit::CandidatePair's in-memory layout, the ccdk_pairs_sink contract)
void launch_keys_to_ids(Ctx& c, const uint64_t* keys, uint64_t n, int nb,
                        const uint8_t* own_kind, const uint32_t* own_index, uint64_t nv,
                        uint64_t ne, uint64_t* ids, int layout = 0, cudaStream_t stream = nullptr);

// Candidate export of ccdk_ccd_into: the final pair list goes to the caller's
// sink from pinned staging, overlapping the narrow phase when possible.
struct PairExport {
    ccdk_pairs_sink sink = nullptr;
    void* user = nullptr;
    bool started = false;
    bool pending = false;  // converted on the device, D2H not yet issued
    uint64_t n = 0;
    void* pin = nullptr;
    int sink_rc = 0;
    std::atomic<bool> aborted { false };
    std::string error;
    std::promise<void> issued; // the worker waits for the D2H to be enqueued
    std::thread worker;
};
// Enqueue the pending export D2H (ccdk_api.cu).  The narrow phase calls it
// right before its generation graph so the bulk copy never sits in front of
// the small pre-narrow copies on the copy engine.
void export_issue(Ctx& c);

// ------------------------------------------------------------------ context

struct Ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::mutex mu;
    uint64_t interval_capacity = 0; // 0 = auto

    DevScene scene;                    // per-call uploads (ccdk_ccd, ccdk_build_boxes, ccdk_classify, ...)
    DevScene resident;                 // ccdk_scene_upload's scene: only the *_resident calls use it
    uint64_t last_nv = 0, last_ne = 0; // id offsets of the scene behind the last pair list

    // boxes / broad phase
    DevBuf bmin, bmax, vids, raw;      // slot order
    DevBuf own_kind, own_index;        // owner of each slot (general mode)
    DevBuf sort_keys_in, sort_keys_out, sort_vals_in, sort_vals_out;
    DevBuf smin_a, smax_a, sbox, svid; // sorted SoA
    DevBuf squant;                     // sorted quantised filter boxes (uint2)
    DevBuf qbounds;                    // quantisation bounds (ordered u32 min[3], max[3])
    DevBuf run_end, seg_off, segs, prefix;
    // slab-mode sweep (K5'): per-box slab counts/offsets, (slab, position)
    // entries before/after the stable slab sort, the slab-major SoA, per-slab
    // segment ends, parameters
    DevBuf slab_cnt, slab_keys, slab_vals, slab_end, slab_par;
    DevBuf emin_a, emax_a, ebox, evid, equant, eslab;
    DevBuf pair_keys, pair_keys_sorted;
    DevBuf rounds;
    DevBuf cub_tmp;
    DevBuf counters;                   // DevCounters
    DevBuf axis;                       // int + reduction partials
    DevBuf partials;
    uint64_t pair_capacity = 0;
    int last_nb = 0;                   // bits per rank in the pair keys
    uint64_t last_n_pairs = 0;
    std::vector<uint64_t> last_rounds;
    bool last_pairs_general = false;

    // queries / narrow phase
    DevBuf q_kind, q_points, q_points_ref, q_sep, q_flags, q_pflags;
    // interval records by split dimension (region) and generation parity
    DevBuf iv_qid[2][3], iv_t[2][3], iv_u[2][3], iv_v[2][3], iv_dep[2][3];
    DevBuf toi_live, toi_snap, splits, exh_gen, zdiag, dirty, out_toi, out_flags;
    DevBuf nscal;                      // NarrowScalars
    GenGraph gen_graph;
    DevBuf gen_sizes;                  // per-generation compacted queue sizes of a run
    PinnedBuf pin_gens;
    std::vector<uint64_t> gen_acc;     // summed over the runs of one narrow phase (exact combined peak)
    bool gen_acc_keep = false;         // chunked callers accumulate across narrow_phase calls
    cudaStream_t copy_stream = nullptr; // H2D of the next chunk while a chunk is narrow-phased
    DevBuf chunk_toi, chunk_flags;     // per-query results gathered over the chunks
    DevBuf chunk_kind, chunk_points, chunk_sep; // the chunk being narrow-phased (fixed addresses)
    int gen_blocks_per_sm = 0;
    uint64_t mem_probe_n = 0;          // narrow interval capacity probed for this many queries
    uint64_t mem_probe_cap = 0;
    EventPool events;
    uint64_t last_query_count = 0;
    uint64_t narrow_launches = 0;
    uint64_t narrow_any_flags = 0;
    // pipeline results across batches
    DevBuf all_keys, all_toi, all_flags;
    bool last_keys_all = false; // fetch_pairs reads all_keys (pipeline) or pair_keys_sorted (API)

    PinnedBuf pin_scene;               // staging of pageable scene uploads
    PinnedBuf pin_axis;                // the broad phase's axis words (read back asynchronously)
    HostPool host_pool;                // helper threads of the staging copies
    // fused classify (K7 into generation 0): records not yet written
    const ClassifySrc* classify_pending = nullptr;
    // candidate export (ccdk_ccd_into)
    PairExport* exp = nullptr;
    DevBuf pair_ids;
    PinnedBuf pin_pairs;

    // staging for API calls
    DevBuf tmp[8];
    PinnedBuf pin;
    PinnedBuf pin_init;                // narrow-phase scalars upload (outlives the async copy)

    // last step results
    DevBuf last_toi;                   // double
};

inline dim3 grid_for(uint64_t n, int block)
{
    uint64_t g = (n + block - 1) / block;
    if (g == 0)
        g = 1;
    if (g > 0x7fffffffULL)
        g = 0x7fffffffULL;
    return dim3(static_cast<unsigned>(g));
}

inline int ceil_log2(uint64_t k)
{
    int b = 1;
    while ((uint64_t(1) << b) < k)
        ++b;
    return b;
}

} // namespace ccdk
