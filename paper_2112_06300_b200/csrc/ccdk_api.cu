// The C ABI (include/ccdk.h): context, validation, the reference-facing entry
// points and the device-resident full CCD step (pipeline.cpp:179-232).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <emmintrin.h>
#include <memory>
#include <thread>

#include "ccdk_internal.cuh"

namespace ccdk {

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(ccdk_ctx* ctx, F&& f)
{
    try {
        f();
        return CCDK_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return CCDK_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return CCDK_CUDA;
    }
    (void)ctx;
}

template <typename T>
T* grow(DevBuf& b, uint64_t n)
{
    return static_cast<T*>(b.ensure(n * sizeof(T)));
}

void h2d(Ctx& c, void* dst, const void* src, size_t bytes)
{
    if (bytes)
        CCDK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.stream));
}

void d2h(Ctx& c, void* dst, const void* src, size_t bytes)
{
    if (bytes)
        CCDK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
}

void sync(Ctx& c) { CCDK_CUDA_CHECK(cudaStreamSynchronize(c.stream)); }

// ---- SceneStep::validate (scene.cpp:13-34) on the device.  Codes follow the
// reference's check order so the first failing check is reported.
enum : unsigned long long {
    kErrNone = ~0ull,
    kErrNonFinite = 1,
    kErrEdgeRange = 2,
    kErrEdgeSame = 3,
    kErrFaceRange = 4,
    kErrFaceSame = 5,
};

const char* scene_error_text(unsigned long long code)
{
    switch (code) {
    case kErrNonFinite:
        return "non-finite vertex coordinate";
    case kErrEdgeRange:
        return "edge index out of range";
    case kErrEdgeSame:
        return "edge endpoints must be distinct";
    case kErrFaceRange:
        return "face index out of range";
    case kErrFaceSame:
        return "face vertices must be distinct";
    }
    return "invalid scene";
}

// The reference throws at the FIRST failing element in its loop order (every
// vertex, then every edge — range before distinctness — then every face), so
// the error key is (element position << 3 | code) and the minimum wins.
__global__ void k_validate_scene(const double* v0, const double* v1, unsigned long long nv,
                                 const uint32_t* e, unsigned long long ne, const uint32_t* f,
                                 unsigned long long nf, unsigned long long* err)
{
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < 3 * nv + ne + nf; i += stride) {
        unsigned long long code = kErrNone, pos = 0;
        if (i < 3 * nv) {
            pos = i / 3; // vertex i/3, coordinate i%3 of both snapshots
            if (!isfinite(v0[i]) || !isfinite(v1[i]))
                code = kErrNonFinite;
        } else if (i < 3 * nv + ne) {
            const unsigned long long j = i - 3 * nv;
            pos = nv + j;
            const uint32_t a = e[2 * j], b = e[2 * j + 1];
            if (a >= nv || b >= nv)
                code = kErrEdgeRange;
            else if (a == b)
                code = kErrEdgeSame;
        } else {
            const unsigned long long j = i - 3 * nv - ne;
            pos = nv + ne + j;
            const uint32_t a = f[3 * j], b = f[3 * j + 1], d = f[3 * j + 2];
            if (a >= nv || b >= nv || d >= nv)
                code = kErrFaceRange;
            else if (a == b || b == d || a == d)
                code = kErrFaceSame;
        }
        if (code != kErrNone)
            atomicMin(err, (pos << 3) | code);
    }
}

// ---- general-box broad phase helpers (arbitrary owners)

__global__ void k_owner_keys(const uint8_t* kind, const uint32_t* index, unsigned long long k,
                             unsigned long long* keys, uint32_t* pos)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= k)
        return;
    keys[i] = (static_cast<unsigned long long>(kind[i]) << 32) | index[i];
    pos[i] = static_cast<uint32_t>(i);
}

__global__ void k_rank_flags(const unsigned long long* skeys, unsigned long long k, uint32_t* flag)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= k)
        return;
    flag[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1u : 0u;
}

// Gather boxes into owner order: SoA corners, vertex triple + rank, raw
// position.  Owner indices are range-checked (the reference's share_vertex
// would index out of bounds).  Ranks are dense over the distinct owners, with
// owner tables by rank (general broad phase), or — canon, run_batched — the
// owner's canonical slot (V, then E, then F), which the pipeline's classify
// and candidate export decode directly; vertex indices must then be < nv.
__global__ void k_gather_general(const float* mn, const float* mx, const uint8_t* kind,
                                 const uint32_t* index, const uint32_t* order,
                                 const uint32_t* rank_incl, unsigned long long k,
                                 unsigned long long nv, const uint32_t* e, unsigned long long ne,
                                 const uint32_t* f, unsigned long long nf, float* bmin,
                                 float* bmax, uint4* vids, uint32_t* raw, uint8_t* own_kind,
                                 uint32_t* own_index, unsigned long long* err, bool canon)
{
    const unsigned long long s = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (s >= k)
        return;
    const unsigned long long r = order[s];
    for (int c = 0; c < 3; ++c) {
        bmin[c * k + s] = mn[3 * r + c];
        bmax[c * k + s] = mx[3 * r + c];
    }
    const uint8_t kd = kind[r];
    const uint32_t ix = index[r];
    uint32_t rank = rank_incl[s] - 1;
    if (canon)
        rank = static_cast<uint32_t>(ix + (kd == CCDK_KIND_EDGE ? nv : kd == CCDK_KIND_FACE ? nv + ne : 0));
    uint4 w = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, rank);
    bool bad = false;
    if (kd == CCDK_KIND_VERTEX) {
        w.x = ix; // share_vertex compares the index itself (scene.cpp:58-60)
        bad = canon && ix >= nv;
    } else if (kd == CCDK_KIND_EDGE) {
        if (ix < ne) {
            w.x = e[2ull * ix];
            w.y = e[2ull * ix + 1];
        } else {
            bad = true;
        }
    } else if (kd == CCDK_KIND_FACE) {
        if (ix < nf) {
            w.x = f[3ull * ix];
            w.y = f[3ull * ix + 1];
            w.z = f[3ull * ix + 2];
        } else {
            bad = true;
        }
    } else {
        bad = true;
    }
    if (bad)
        atomicMin(err, s);
    vids[s] = w;
    raw[s] = static_cast<uint32_t>(r);
    if (!canon) {
        own_kind[rank] = kd;
        own_index[rank] = ix;
    }
}

__global__ void k_aos_to_soa(const float* mn, const float* mx, unsigned long long k, float* bmin,
                             float* bmax)
{
    const unsigned long long s = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (s >= k)
        return;
    for (int c = 0; c < 3; ++c) {
        bmin[c * k + s] = mn[3 * s + c];
        bmax[c * k + s] = mx[3 * s + c];
    }
}

// ---- classify over arbitrary pair lists (broadphase.cpp:194-239)
__global__ void k_classify_flags(const unsigned long long* pairs, unsigned long long n,
                                 unsigned long long nv, const uint32_t* e, unsigned long long ne,
                                 const uint32_t* f, unsigned long long nf, uint32_t* fvf,
                                 uint32_t* fee, unsigned long long* err)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    const unsigned long long a = pairs[2 * i], b = pairs[2 * i + 1];
    const unsigned ka = static_cast<unsigned>(a >> 32), kb = static_cast<unsigned>(b >> 32);
    const uint32_t ia = static_cast<uint32_t>(a), ib = static_cast<uint32_t>(b);
    const auto limit = [&](unsigned kd) { return kd == 0 ? nv : kd == 1 ? ne : nf; };
    uint32_t vf = 0, ee = 0;
    if (ka > 2 || kb > 2 || ia >= limit(ka) || ib >= limit(kb)) {
        atomicMin(err, i);
    } else if (ka == CCDK_KIND_VERTEX && kb == CCDK_KIND_FACE) {
        vf = (ia != f[3ull * ib] && ia != f[3ull * ib + 1] && ia != f[3ull * ib + 2]) ? 1u : 0u;
    } else if (ka == CCDK_KIND_EDGE && kb == CCDK_KIND_EDGE) {
        const uint32_t a0 = e[2ull * ia], a1 = e[2ull * ia + 1], b0 = e[2ull * ib], b1 = e[2ull * ib + 1];
        ee = (a0 != b0 && a0 != b1 && a1 != b0 && a1 != b1) ? 1u : 0u;
    }
    fvf[i] = vf;
    fee[i] = ee;
}

__global__ void k_classify_write(const unsigned long long* pairs, unsigned long long n,
                                 const uint32_t* fvf, const uint32_t* fee, const uint32_t* ovf,
                                 const uint32_t* oee, const unsigned long long* n_vf_ptr,
                                 const double* v0, const double* v1, const uint32_t* e,
                                 const uint32_t* f, uint8_t* kind, double* pts,
                                 unsigned long long* src)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n || !(fvf[i] | fee[i]))
        return;
    const unsigned long long a = pairs[2 * i], b = pairs[2 * i + 1];
    const uint32_t ia = static_cast<uint32_t>(a), ib = static_cast<uint32_t>(b);
    uint32_t pv[4];
    unsigned long long q;
    if (fvf[i]) {
        q = ovf[i];
        pv[0] = ia;
        pv[1] = f[3ull * ib];
        pv[2] = f[3ull * ib + 1];
        pv[3] = f[3ull * ib + 2];
        kind[q] = CCDK_QUERY_VF;
    } else {
        q = *n_vf_ptr + oee[i];
        pv[0] = e[2ull * ia];
        pv[1] = e[2ull * ia + 1];
        pv[2] = e[2ull * ib];
        pv[3] = e[2ull * ib + 1];
        kind[q] = CCDK_QUERY_EE;
    }
    for (int p = 0; p < 4; ++p)
        for (int c = 0; c < 3; ++c) {
            pts[24 * q + 3 * p + c] = v0[3ull * pv[p] + c];
            pts[24 * q + 12 + 3 * p + c] = v1[3ull * pv[p] + c];
        }
    src[2 * q] = a;
    src[2 * q + 1] = b;
}

__global__ void k_count_total(const uint32_t* flags, const uint32_t* offs, unsigned long long n,
                              unsigned long long* out)
{
    *out = n ? static_cast<unsigned long long>(offs[n - 1]) + flags[n - 1] : 0;
}

__global__ void k_count_vf(const unsigned long long* keys, unsigned long long n, int nb,
                           unsigned long long nv, unsigned long long* out)
{
    // keys are sorted: VF keys (lo rank < nv) form a prefix
    unsigned long long a = 0, b = n;
    while (a < b) {
        const unsigned long long m = (a + b) >> 1;
        if ((keys[m] >> nb) < nv)
            a = m + 1;
        else
            b = m;
    }
    *out = a;
}

__global__ void k_store_toi(const NarrowScalars* sc, int have_queries, double* out)
{
    *out = have_queries ? __longlong_as_double(static_cast<long long>(sc->global_toi_bits))
                        : CUDART_INF;
}

template <typename F>
void cub_call(Ctx& c, F&& f)
{
    size_t bytes = 0;
    CCDK_CUDA_CHECK(f(nullptr, bytes));
    void* tmp = c.cub_tmp.ensure(bytes);
    CCDK_CUDA_CHECK(f(tmp, bytes));
}

void validate_narrow_cfg(const ccdk_narrow_cfg& c)
{
    // NarrowConfig::validate, narrowphase.cpp:10-20
    if (!(c.delta > 0.0))
        throw Error(CCDK_CONFIG, "NarrowConfig: delta must be > 0");
    if (c.max_splits < 1)
        throw Error(CCDK_CONFIG, "NarrowConfig: max_splits must be >= 1");
    if (c.min_separation < 0.0)
        throw Error(CCDK_CONFIG, "NarrowConfig: min_separation must be >= 0");
    if (!(c.t_max > 0.0) || c.t_max > 1.0)
        throw Error(CCDK_CONFIG, "NarrowConfig: t_max must be in (0, 1]");
}

void validate_pipeline_cfg(const ccdk_pipeline_cfg& p)
{
    // PipelineConfig::validate, pipeline.cpp:23-37
    validate_narrow_cfg(p.narrow);
    if (p.rs_params == 0 || p.rs_query == 0 || p.rs_interval == 0 || p.rs_pair_ints == 0)
        throw Error(CCDK_CONFIG, "PipelineConfig: record sizes must be positive");
    if (p.memory_budget <= p.rs_params)
        throw Error(CCDK_CONFIG, "PipelineConfig: memory budget must exceed the parameter size");
    if (p.min_sep_fraction < 0.0)
        throw Error(CCDK_CONFIG, "PipelineConfig: min_sep_fraction must be >= 0");
    if (p.threads < 1)
        throw Error(CCDK_CONFIG, "PipelineConfig: threads must be >= 1");
    if (p.inflation < 0.0)
        throw Error(CCDK_CONFIG, "PipelineConfig: inflation must be >= 0");
}

void validate_scene_dev(Ctx& c, DevScene& s)
{
    auto* ctr = static_cast<DevCounters*>(c.counters.ensure(sizeof(DevCounters)));
    CCDK_CUDA_CHECK(cudaMemsetAsync(&ctr->misc[3], 0xff, 8, c.stream));
    const uint64_t n = 3 * s.nv + s.ne + s.nf;
    if (n) {
        k_validate_scene<<<std::min<unsigned>(grid_for(n, 256).x, 8u * c.num_sms), 256, 0, c.stream>>>(
            s.v0.as<double>(), s.v1.as<double>(), s.nv, s.edges.as<uint32_t>(), s.ne,
            s.faces.as<uint32_t>(), s.nf, &ctr->misc[3]);
        CCDK_LAUNCH_CHECK();
    }
}

void check_scene_error(Ctx& c)
{
    auto* ctr = c.counters.as<DevCounters>();
    unsigned long long code = 0;
    d2h(c, &code, &ctr->misc[3], 8);
    sync(c);
    if (code != kErrNone)
        throw Error(CCDK_INVALID_INPUT, scene_error_text(code & 7));
}

// Host -> device copies of a scene's arrays.  Pinned sources go straight to
// the DMA engine.  Pageable sources (ordinary std::vector storage, the
// drop-in's case) are copied by the host into the context's pinned staging
// buffer in 1 MB chunks, several threads at once for large scenes, and each
// chunk's DMA is enqueued as soon as it is staged — the host copy and the
// transfer overlap instead of the driver's serial pageable path (measured
// ~10 GB/s for a 16 MB scene).  The staging stores are non-temporal: with
// ordinary stores the host's memory bandwidth, shared by the copy's reads,
// writes and read-for-ownership and the DMA's reads, held the 16 MB C4
// upload at 1.1 ms; streaming stores take it to 0.5 ms (tools/upload_sweep.sh).
struct HostPiece {
    void* dst;
    const void* src;
    size_t bytes;
};

bool is_pinned(const void* p)
{
    cudaPointerAttributes at {};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError(); // unregistered memory on older runtimes: clear the error
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Copy into pinned staging with non-temporal stores: the staging lines are
// read next by the DMA engine, not the CPU, so skipping the read-for-ownership
// saves a third of the host memory traffic of the copy (dst 16-byte aligned).
void stream_copy(void* dst, const void* src, size_t n)
{
    if (reinterpret_cast<uintptr_t>(dst) & 15) {
        std::memcpy(dst, src, n);
        return;
    }
    auto* d = static_cast<__m128i*>(dst);
    const auto* s = static_cast<const __m128i*>(src);
    const size_t v = n / 16;
    for (size_t i = 0; i < v; i += 4) {
        if (i + 4 <= v) {
            const __m128i a = _mm_loadu_si128(s + i), b = _mm_loadu_si128(s + i + 1);
            const __m128i e = _mm_loadu_si128(s + i + 2), f = _mm_loadu_si128(s + i + 3);
            _mm_stream_si128(d + i, a);
            _mm_stream_si128(d + i + 1, b);
            _mm_stream_si128(d + i + 2, e);
            _mm_stream_si128(d + i + 3, f);
        } else {
            for (size_t j = i; j < v; ++j)
                _mm_stream_si128(d + j, _mm_loadu_si128(s + j));
        }
    }
    std::memcpy(static_cast<char*>(dst) + 16 * v, static_cast<const char*>(src) + 16 * v, n - 16 * v);
    _mm_sfence();
}

size_t env_size(const char* name, size_t dflt)
{
    const char* v = std::getenv(name);
    return v && *v ? static_cast<size_t>(std::strtoull(v, nullptr, 10)) : dflt;
}

void upload_pieces(Ctx& c, const HostPiece* pieces, int n)
{
    // staging chunk and helper count (CCDK_STAGE_CHUNK_KB / CCDK_STAGE_THREADS: A/B switches)
    static const size_t kChunk = env_size("CCDK_STAGE_CHUNK_KB", 1024) << 10;
    static const size_t kMaxHelpers = env_size("CCDK_STAGE_THREADS", 7);
    static const bool kStream = env_size("CCDK_STAGE_NT", 1) != 0;
    size_t staged = 0;
    struct Chunk {
        void* dst;
        const void* src;
        size_t bytes, off;
    };
    std::vector<Chunk> chunks;
    for (int i = 0; i < n; ++i) {
        const HostPiece& pc = pieces[i];
        if (!pc.bytes)
            continue;
        if (pc.bytes < kChunk || is_pinned(pc.src)) {
            h2d(c, pc.dst, pc.src, pc.bytes); // small or already pinned
            continue;
        }
        for (size_t o = 0; o < pc.bytes; o += kChunk) {
            const size_t b = std::min(kChunk, pc.bytes - o);
            chunks.push_back({ static_cast<char*>(pc.dst) + o, static_cast<const char*>(pc.src) + o, b, staged });
            staged += (b + 63) & ~size_t(63); // staging slots 64-byte aligned (streaming stores)
        }
    }
    if (chunks.empty())
        return;
    char* pin = static_cast<char*>(c.pin_scene.ensure(staged));
    // the context's helper threads and the caller each copy a chunk into
    // pinned staging and enqueue its DMA (measured faster than funnelling
    // every DMA through the caller)
    std::atomic<size_t> next { 0 };
    std::atomic<int> failed { 0 };
    const int device = c.device;
    static const bool trace = std::getenv("CCDK_UPLOAD_TRACE") != nullptr;
    using TClock = std::chrono::steady_clock;
    const auto t0 = TClock::now();
    std::vector<double> tr(trace ? 3 * chunks.size() : 0);
    auto us = [&] { return std::chrono::duration<double, std::micro>(TClock::now() - t0).count(); };
    auto work = [&, device] {
        cudaSetDevice(device); // helper threads start on device 0
        for (size_t k; (k = next.fetch_add(1)) < chunks.size();) {
            const Chunk& ch = chunks[k];
            if (trace)
                tr[3 * k] = us();
            if (kStream)
                stream_copy(pin + ch.off, ch.src, ch.bytes);
            else
                std::memcpy(pin + ch.off, ch.src, ch.bytes);
            if (trace)
                tr[3 * k + 1] = us();
            if (cudaMemcpyAsync(ch.dst, pin + ch.off, ch.bytes, cudaMemcpyHostToDevice, c.stream) != cudaSuccess)
                failed = 1;
            if (trace)
                tr[3 * k + 2] = us();
        }
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned helpers = static_cast<unsigned>(std::min<size_t>({ kMaxHelpers, hw / 2, chunks.size() / 2 }));
    cudaEvent_t ev[2] = { nullptr, nullptr };
    if (trace) {
        cudaEventCreate(&ev[0]);
        cudaEventCreate(&ev[1]);
        cudaEventRecord(ev[0], c.stream);
    }
    c.host_pool.run(work, helpers);
    if (trace) { // diagnostics: per chunk (copy start, copy end, DMA enqueued) in us
        cudaEventRecord(ev[1], c.stream);
        cudaEventSynchronize(ev[1]);
        float gms = 0;
        cudaEventElapsedTime(&gms, ev[0], ev[1]);
        fprintf(stderr, "[ccdk upload] stream %.0f us, host sync at %.0f us; ", 1000 * gms, us());
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        fprintf(stderr, "%zu chunks, %u helpers:", chunks.size(), helpers);
        for (size_t k = 0; k < chunks.size(); ++k)
            fprintf(stderr, " (%.0f %.0f %.0f)", tr[3 * k], tr[3 * k + 1], tr[3 * k + 2]);
        fprintf(stderr, " returned %.0f\n", us());
    }
    if (failed)
        CCDK_CUDA_CHECK(cudaGetLastError());
}

// Upload a scene into a context slot (per-call scratch or the resident
// scene) and validate it on the device (SceneStep::validate,
// scene.cpp:13-34) before any kernel indexes it.
void upload_scene(Ctx& c, DevScene& s, const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                  uint64_t ne, const uint32_t* f, uint64_t nf)
{
    s.valid = false;
    s.nv = nv;
    s.ne = ne;
    s.nf = nf;
    const HostPiece pieces[4] = { { s.v0.ensure(nv * 24), v0, nv * 24 },
                                  { s.v1.ensure(nv * 24), v1, nv * 24 },
                                  { s.edges.ensure(ne * 8), e, ne * 8 },
                                  { s.faces.ensure(nf * 12), f, nf * 12 } };
    static const bool trace = std::getenv("CCDK_UPLOAD_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    upload_pieces(c, pieces, 4);
    if (trace)
        sync(c);
    const auto t1 = std::chrono::steady_clock::now();
    validate_scene_dev(c, s);
    check_scene_error(c);
    if (trace) // diagnostics: exposed upload and validation time
        fprintf(stderr, "[ccdk upload] %.3f ms copies, %.3f ms validation\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    s.valid = true;
}

// ---- candidate export (ccdk_ccd_into).  The final canonical key list is
// converted to ccdkit::CandidatePair's layout on the device, copied into
// pinned staging on the copy stream, and handed to the caller's sink — on a
// worker thread while the compute stream runs classify + narrow phase (single
// broad batch), or inline at the end of the step (batched steps).
void export_begin(Ctx& c, const uint64_t* keys, uint64_t n, uint64_t nv, uint64_t ne, bool async)
{
    PairExport& x = *c.exp;
    x.started = true;
    x.n = n;
    if (!c.copy_stream)
        CCDK_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    x.pin = c.pin_pairs.ensure(std::max<uint64_t>(16 * n, 16));
    if (n)
        launch_keys_to_ids(c, keys, n, c.last_nb, nullptr, nullptr, nv, ne, grow<uint64_t>(c.pair_ids, 2 * n), 1);
    x.pending = true;
    cudaEvent_t done = c.events.get(EventPool::kExport + 1);
    const int device = c.device;
    auto deliver = [&x, done, device](std::shared_future<void> issued) {
        // announce the count first: the caller allocates (and faults in) its
        // destination while the copy is still in flight
        x.sink_rc = x.sink(x.user, nullptr, x.n);
        issued.wait();
        if (x.sink_rc || x.aborted.load())
            return;
        cudaSetDevice(device);
        const cudaError_t r = cudaEventSynchronize(done);
        if (r != cudaSuccess) {
            x.error = std::string("candidate export: ") + cudaGetErrorString(r);
            return;
        }
        x.sink_rc = x.sink(x.user, static_cast<const uint64_t*>(x.pin), x.n);
    };
    std::shared_future<void> issued = x.issued.get_future().share();
    if (async) {
        x.worker = std::thread(deliver, issued);
    } else {
        export_issue(c);
        deliver(issued);
    }
}

} // namespace

void export_issue(Ctx& c)
{
    PairExport& x = *c.exp;
    if (!x.pending)
        return;
    x.pending = false;
    cudaEvent_t ready = c.events.get(EventPool::kExport), done = c.events.get(EventPool::kExport + 1);
    try {
        if (x.n) {
            CCDK_CUDA_CHECK(cudaEventRecord(ready, c.stream));
            CCDK_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, ready, 0));
            CCDK_CUDA_CHECK(cudaMemcpyAsync(x.pin, c.pair_ids.as<uint64_t>(), 16 * x.n, cudaMemcpyDeviceToHost,
                                            c.copy_stream));
        }
        CCDK_CUDA_CHECK(cudaEventRecord(done, c.copy_stream));
    } catch (...) {
        x.issued.set_value();
        throw;
    }
    x.issued.set_value();
}

namespace {

void export_finish(Ctx& c)
{
    PairExport& x = *c.exp;
    export_issue(c); // no narrow phase ran (no candidates): issue now
    if (x.worker.joinable())
        x.worker.join();
    if (!x.error.empty())
        throw Error(CCDK_CUDA, x.error);
    if (x.sink_rc)
        throw Error(CCDK_OOM, "ccdk_ccd_into: the candidate sink failed");
}

// A caller's box list on the device in owner order (slot order = the sort's
// tie-break, broadphase.cpp:22-34): upload, sort by owner, gather.  Owners
// are range-checked here (one round trip); nranks < k means duplicate owners.
struct UserBoxes {
    float* bmin = nullptr;
    float* bmax = nullptr;
    uint4* vids = nullptr;
    uint32_t* raw = nullptr;
    uint64_t nranks = 0;
};

// run_batched's box list as the caller holds it (host AoS split into arrays)
struct HostBoxes {
    const float* min_corner = nullptr; // [k][3]
    const float* max_corner = nullptr;
    const uint8_t* owner_kind = nullptr;
    const uint32_t* owner_index = nullptr;
    uint64_t k = 0;
};

UserBoxes gather_user_boxes(Ctx& c, const float* min_corner, const float* max_corner, const uint8_t* owner_kind,
                            const uint32_t* owner_index, uint64_t k, uint64_t nv, const uint32_t* e, uint64_t ne,
                            const uint32_t* f, uint64_t nf, bool canon, const char* what)
{
    cudaStream_t s = c.stream;
    float* mn = grow<float>(c.tmp[0], 3 * k);
    float* mx = grow<float>(c.tmp[1], 3 * k);
    uint8_t* kd = grow<uint8_t>(c.tmp[2], k);
    uint32_t* ix = grow<uint32_t>(c.tmp[3], k);
    h2d(c, mn, min_corner, 12 * k);
    h2d(c, mx, max_corner, 12 * k);
    h2d(c, kd, owner_kind, k);
    h2d(c, ix, owner_index, 4 * k);
    // owner order + dense ranks
    unsigned long long* okeys = grow<unsigned long long>(c.tmp[4], 2 * k);
    uint32_t* pos = grow<uint32_t>(c.tmp[5], 2 * k);
    k_owner_keys<<<grid_for(k, 256), 256, 0, s>>>(kd, ix, k, okeys, pos);
    CCDK_LAUNCH_CHECK();
    cub_call(c, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, okeys, okeys + k, pos, pos + k, static_cast<int64_t>(k), 0, 34,
                                               s);
    });
    uint32_t* flag = grow<uint32_t>(c.tmp[6], 2 * k);
    k_rank_flags<<<grid_for(k, 256), 256, 0, s>>>(okeys + k, k, flag);
    cub_call(c, [&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, flag, flag + k, static_cast<int64_t>(k), s);
    });
    UserBoxes ub;
    ub.bmin = grow<float>(c.bmin, 3 * k);
    ub.bmax = grow<float>(c.bmax, 3 * k);
    ub.vids = grow<uint4>(c.vids, k);
    ub.raw = grow<uint32_t>(c.raw, 2 * k);
    uint8_t* own_kind = grow<uint8_t>(c.own_kind, k);
    uint32_t* own_index = grow<uint32_t>(c.own_index, k);
    auto* ctr = static_cast<DevCounters*>(c.counters.ensure(sizeof(DevCounters)));
    CCDK_CUDA_CHECK(cudaMemsetAsync(&ctr->error, 0xff, 8, s));
    k_gather_general<<<grid_for(k, 256), 256, 0, s>>>(mn, mx, kd, ix, pos + k, flag + k, k, nv, e, ne, f, nf,
                                                      ub.bmin, ub.bmax, ub.vids, ub.raw, own_kind, own_index,
                                                      &ctr->error, canon);
    CCDK_LAUNCH_CHECK();
    uint32_t nranks = 0;
    unsigned long long err = 0;
    d2h(c, &nranks, flag + 2 * k - 1, 4);
    d2h(c, &err, &ctr->error, 8);
    sync(c);
    if (err != ~0ull)
        throw Error(CCDK_INVALID_INPUT, std::string(what) + ": box owner index out of range");
    ub.nranks = nranks;
    return ub;
}

// run_batched's BatchRun (pipeline.cpp:81-175) over device primitives.  The
// recursion structure, capacities and counters follow the reference so the
// batch count and tracked bytes agree; every broad/narrow batch is a device
// run.  At the default budget this is exactly one broad and one narrow batch.
struct BatchRun {
    Ctx& c;
    const ccdk_pipeline_cfg& cfg;
    DevScene& s;
    uint64_t k;
    uint64_t cap_pairs;
    float* bmin = nullptr;
    float* bmax = nullptr;
    uint4* vids = nullptr;
    unsigned long long toi_bits = 0x7ff0000000000000ull;
    bool tol = false, zd = false;
    uint64_t candidates = 0, queries = 0, vf = 0, narrow_batches = 0, broad_batches = 0;
    uint64_t pair_tests = 0, total_splits = 0, evaluations = 0, split_actions = 0;
    uint64_t generations = 0, peak_queue = 0, launches = 0;
    uint64_t peak_bytes = 0, base_bytes = 0;
    float ms_sort = 0, ms_sweep = 0, ms_pairsort = 0, ms_classify = 0, ms_narrow = 0;
    int axis = 0;
    uint64_t slabs = 0, slab_entries = 0;
    bool check_build_error = false; // the box build's flag, checked by the first broad phase
    // a caller's box list (run_batched): raw input positions, duplicate
    // owners, ranks = canonical slots over rank_bits
    const uint32_t* raw = nullptr;
    bool unique = false;
    int rank_bits = 0;

    // broad_batch (pipeline.cpp:140-174): halve the sweep range while the
    // candidates exceed the budget's pair capacity
    void broad_batch(uint64_t begin, uint64_t end, uint32_t shard_rank = 0, uint32_t shard_count = 1,
                     bool allow_slab = true)
    {
        BroadIn bi;
        bi.bmin = bmin;
        bi.bmax = bmax;
        bi.vids = vids;
        bi.k = k;
        bi.raw = raw;
        bi.unique = unique;
        bi.rank_bits = rank_bits;
        bi.range_begin = begin;
        bi.range_end = end;
        bi.shard_rank = shard_rank;
        bi.shard_count = shard_count;
        // the axis matters only if the budget can force range halving
        bi.exact_axis = cap_pairs < k * (k - 1) / 2;
        // stq/sap/bf give the identical set; the halved ranges differ: bf
        // splits raw box positions, stq/sap sorted ones (pipeline.cpp:65-77)
        bi.method = cfg.broad_method == CCDK_BROAD_BF && bi.exact_axis && shard_count == 1 ? CCDK_BROAD_BF
                                                                                          : CCDK_BROAD_STQ;
        bi.allow_slab = allow_slab;
        bi.check_build_error = check_build_error;
        check_build_error = false; // checked at this broad phase's first read-back
        bi.defer_collect = true;   // times / axis read after the narrow phase's own sync
        BroadOut bo;
        broad_phase(c, bi, bo);
        launches += bo.launches;
        pair_tests += bo.pair_tests;
        slabs = bo.slab_count;
        slab_entries = bo.slab_entries;
        auto collect = [&] {
            broad_collect(c, bo);
            ms_sort += bo.ms_axis_sort;
            ms_sweep += bo.ms_sweep;
            ms_pairsort += bo.ms_pairsort;
            axis = bo.axis;
        };
        if (shard_count > 1 && bo.slab_mode && bo.n_pairs > cap_pairs) {
            // budget halving is defined on sorted positions: redo this shard 1-D
            collect();
            broad_batch(begin, end, shard_rank, shard_count, false);
            return;
        }
        if (shard_count > 1) { // this shard's slice of sorted left positions
            begin = bo.range_lo;
            end = bo.range_hi;
        }
        if (bo.n_pairs > cap_pairs && end - begin > 1) {
            collect(); // before the next broad phase reuses the events
            const uint64_t mid = begin + (end - begin) / 2;
            broad_batch(begin, mid);
            broad_batch(mid, end);
            return;
        }
        // the whole step in one broad batch: these keys are the final list
        if (c.exp && !c.exp->started && broad_batches == 0 && begin == 0 && end >= k && shard_count == 1)
            export_begin(c, c.pair_keys_sorted.as<uint64_t>(), bo.n_pairs, s.nv, s.ne, true);
        ++broad_batches;
        process_keys(c.pair_keys_sorted.as<uint64_t>(), bo.n_pairs);
        collect();
    }

    // The rest of a broad batch on canonical pair keys (lo << nb | hi over
    // slot ranks): append them to the step's candidate list, classify
    // (K7) + query_min_separations, narrow phase.  Also the entry for keys
    // supplied from outside (multi-GPU rebalance).
    void process_keys(const uint64_t* keys, uint64_t n)
    {
        uint64_t* all = static_cast<uint64_t*>(c.all_keys.ensure_keep((candidates + n) * 8, c.stream));
        if (n)
            CCDK_CUDA_CHECK(cudaMemcpyAsync(all + candidates, keys, n * 8, cudaMemcpyDeviceToDevice, c.stream));
        candidates += n;
        base_bytes = k * 32 + candidates * 16;
        // classify (K7) + query_min_separations
        cudaEvent_t e0 = c.events.get(EventPool::kBatch), e1 = c.events.get(EventPool::kBatch + 1);
        CCDK_CUDA_CHECK(cudaEventRecord(e0, c.stream));
        uint8_t* qk = grow<uint8_t>(c.q_kind, std::max<uint64_t>(n, 1));
        double* qp = grow<double>(c.q_points, 24 * std::max<uint64_t>(n, 1));
        uint32_t* qfl = grow<uint32_t>(c.q_pflags, std::max<uint64_t>(n, 1));
        // K7: fused into the narrow phase's generation 0 (k_classify_gen0)
        // unless the per-query separations need the records first
        ClassifySrc src;
        src.keys = keys;
        src.n = n;
        src.nb = c.last_nb;
        src.v0 = s.v0.as<double>();
        src.v1 = s.v1.as<double>();
        src.nv = s.nv;
        src.e = s.edges.as<uint32_t>();
        src.ne = s.ne;
        src.f = s.faces.as<uint32_t>();
        src.kind_out = qk;
        src.pts_out = qp;
        src.qflags_out = qfl;
        static const bool no_fuse_classify = std::getenv("CCDK_NO_FUSE_CLASSIFY") != nullptr;
        const bool fuse_classify = n && !no_fuse_classify && cfg.min_sep_mode != CCDK_MINSEP_RELATIVE;
        struct Pending { // never leave a dangling pending classification
            Ctx& c;
            ~Pending() { c.classify_pending = nullptr; }
        } pending_guard { c };
        if (fuse_classify)
            c.classify_pending = &src;
        else
            launch_classify_keys(c, keys, n, c.last_nb, s.v0.as<double>(), s.v1.as<double>(), s.nv,
                                 s.edges.as<uint32_t>(), s.ne, s.faces.as<uint32_t>(), qk, qp, qfl);
        double* seps = nullptr;
        if (cfg.min_sep_mode == CCDK_MINSEP_RELATIVE && n) {
            seps = grow<double>(c.q_sep, n);
            launch_min_seps(c, qk, qp, n, cfg, seps, true);
            ++launches;
        }
        // the VF count goes to pinned memory and is read after the narrow
        // phase's own sync (a pageable read-back here would drain the queue
        // before the narrow phase is even enqueued)
        unsigned long long* nvf_h = static_cast<unsigned long long*>(c.pin_axis.ensure(64)) + 4;
        *nvf_h = 0;
        if (n) {
            auto* ctr = c.counters.as<DevCounters>();
            k_count_vf<<<1, 1, 0, c.stream>>>(reinterpret_cast<const unsigned long long*>(keys), n,
                                              c.last_nb, s.nv, &ctr->misc[2]);
            CCDK_LAUNCH_CHECK();
            d2h(c, nvf_h, &ctr->misc[2], 8);
            launches += 2;
        }
        CCDK_CUDA_CHECK(cudaEventRecord(e1, c.stream));
        const uint64_t qoff = queries;
        queries += n;
        grow_results(queries);
        if (n)
            narrow_batch(qk, qp, seps, qfl, 0, n, qoff);
        else
            ++narrow_batches; // an empty narrow run still counts as a batch
        ensure_classified(c); // the records exist after the step whatever path ran
        CCDK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0;
        CCDK_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        ms_classify += ms;
        vf += *nvf_h;
    }

    void grow_results(uint64_t nq)
    {
        c.all_toi.ensure_keep(std::max<uint64_t>(nq, 1) * 8, c.stream);
        c.all_flags.ensure_keep(std::max<uint64_t>(nq, 1), c.stream);
    }

    // narrow_batch (pipeline.cpp:103-138): queue capacity from the budget,
    // halve the queries on overflow
    void narrow_batch(const uint8_t* qk, const double* qp, const double* seps, const uint32_t* qfl,
                      uint64_t lo, uint64_t hi, uint64_t qoff)
    {
        const uint64_t n_sub = hi - lo;
        const uint64_t pair_bytes = n_sub * (cfg.rs_query + 3 * cfg.rs_pair_ints);
        const uint64_t avail = cfg.memory_budget > cfg.rs_params + pair_bytes
            ? cfg.memory_budget - cfg.rs_params - pair_bytes
            : 0;
        NarrowIn ni;
        ni.kind = qk + lo;
        ni.points = qp + 24 * lo;
        ni.sep = seps ? seps + lo : nullptr;
        ni.qflags = qfl ? qfl + lo : nullptr;
        ni.n = n_sub;
        ni.cfg = cfg.narrow;
        ni.queue_capacity = avail / cfg.rs_interval;
        NarrowOut no;
        narrow_phase(c, ni, no);
        launches += 2 + no.launches;
        ms_narrow += static_cast<float>(no.stats.device_ms);
        if (no.stats.overflow) {
            if (n_sub <= 1)
                throw Error(CCDK_CONFIG, "memory budget too small to hold even one query");
            const uint64_t mid = lo + n_sub / 2;
            narrow_batch(qk, qp, seps, qfl, lo, mid, qoff);
            narrow_batch(qk, qp, seps, qfl, mid, hi, qoff);
            return;
        }
        ++narrow_batches;
        const unsigned long long gb = static_cast<unsigned long long>(
            __builtin_bit_cast(uint64_t, no.stats.global_toi));
        toi_bits = std::min(toi_bits, gb);
        tol = tol || (no.any_flags & CCDK_FLAG_TOLERANCE_HIT);
        zd = zd || (no.any_flags & CCDK_FLAG_ZERO_TOI_DIAG);
        total_splits += no.stats.total_splits;
        evaluations += no.stats.evaluations;
        split_actions += no.stats.split_actions;
        generations = std::max<uint64_t>(generations, no.stats.generations);
        peak_queue = std::max<uint64_t>(peak_queue, no.stats.peak_queue);
        CCDK_CUDA_CHECK(cudaMemcpyAsync(c.all_toi.as<double>() + qoff + lo, no.toi, 8 * n_sub,
                                        cudaMemcpyDeviceToDevice, c.stream));
        CCDK_CUDA_CHECK(cudaMemcpyAsync(c.all_flags.as<uint8_t>() + qoff + lo, no.flags, n_sub,
                                        cudaMemcpyDeviceToDevice, c.stream));
        peak_bytes = std::max<uint64_t>(peak_bytes, base_bytes + n_sub * 216 + no.stats.peak_queue * 216);
    }
};

void finish_step(Ctx& c, DevScene& s, BatchRun& run, uint64_t k, ccdk_report& rep, cudaEvent_t start_event,
                 cudaEvent_t* ev);

// The full CCD step on ctx.scene (pipeline.cpp:218-232 via run_batched at the
// default budget): build -> STQ -> classify -> narrow -> global min.
void ccd_step(Ctx& c, DevScene& s, const ccdk_pipeline_cfg& cfg, uint32_t shard_rank, uint32_t shard_count,
              ccdk_report& rep, cudaEvent_t start_event, const HostBoxes* hb = nullptr)
{
    validate_pipeline_cfg(cfg);
    std::memset(&rep, 0, sizeof rep);
    rep.toi = INFINITY;
    rep.batch_count = 1;
    const uint64_t k = hb ? hb->k : s.nv + s.ne + s.nf;
    cudaStream_t st = c.stream;
    // run_batched (pipeline.cpp:184-187): candidate capacity of the budget
    const uint64_t cap_pairs = (cfg.memory_budget - cfg.rs_params) / (cfg.rs_query + 3 * cfg.rs_pair_ints);
    if (cap_pairs < 1)
        throw Error(CCDK_CONFIG, "memory budget too small to hold even one query");
    cudaEvent_t ev[6];
    for (int i = 0; i < 6; ++i)
        ev[i] = c.events.get(EventPool::kStep + i);
    CCDK_CUDA_CHECK(cudaEventRecord(ev[0], st));

    if (hb) { // run_batched on the caller's boxes: no K1
        BatchRun run { c, cfg, s, k, cap_pairs };
        if (k) {
            const UserBoxes ub = gather_user_boxes(c, hb->min_corner, hb->max_corner, hb->owner_kind,
                                                   hb->owner_index, k, s.nv, s.edges.as<uint32_t>(), s.ne,
                                                   s.faces.as<uint32_t>(), s.nf, true, "run_batched");
            CCDK_CUDA_CHECK(cudaEventRecord(ev[1], st));
            run.bmin = ub.bmin;
            run.bmax = ub.bmax;
            run.vids = ub.vids;
            run.raw = ub.raw;
            run.unique = ub.nranks < k;
            run.rank_bits = ceil_log2(std::max<uint64_t>(s.nv + s.ne + s.nf, 2));
            run.broad_batch(0, k, shard_rank, shard_count);
        } else {
            CCDK_CUDA_CHECK(cudaEventRecord(ev[1], st));
            run.narrow_batches = 1;
        }
        finish_step(c, s, run, k, rep, start_event, ev);
        return;
    }
    // K1 (the scene was validated when it was uploaded)
    float* bmin = grow<float>(c.bmin, 3 * std::max<uint64_t>(k, 1));
    float* bmax = grow<float>(c.bmax, 3 * std::max<uint64_t>(k, 1));
    uint4* vids = grow<uint4>(c.vids, std::max<uint64_t>(k, 1));
    launch_build_boxes(c, s.v0.as<double>(), s.v1.as<double>(), s.nv, s.edges.as<uint32_t>(), s.ne,
                       s.faces.as<uint32_t>(), s.nf, cfg.inflation, bmin, bmax, vids);
    CCDK_CUDA_CHECK(cudaEventRecord(ev[1], st));
    if (k && k < 2) { // no broad phase to fold the check into
        auto* ctr = c.counters.as<DevCounters>();
        unsigned long long err = 0;
        d2h(c, &err, &ctr->error, 8);
        sync(c);
        if (err != ~0ull)
            throw Error(CCDK_INVALID_INPUT, "round_down_reduced: non-finite input");
    }
    BatchRun run { c, cfg, s, k, cap_pairs };
    run.check_build_error = k >= 2; // at the broad phase's first read-back (one round trip fewer)
    run.bmin = bmin;
    run.bmax = bmax;
    run.vids = vids;
    if (k)
        run.broad_batch(0, k, shard_rank, shard_count);
    else
        run.narrow_batches = 1;
    finish_step(c, s, run, k, rep, start_event, ev);
}

// The step's tail: the candidate union in canonical order, the export, the
// report (pipeline.cpp:196-214).
void finish_step(Ctx& c, DevScene& s, BatchRun& run, uint64_t k, ccdk_report& rep, cudaEvent_t start_event,
                 cudaEvent_t* ev)
{
    cudaStream_t st = c.stream;
    // canonical order of the candidate union across batches (pipeline.cpp:196)
    if (run.broad_batches > 1 && run.candidates) {
        uint64_t* all = c.all_keys.as<uint64_t>();
        uint64_t* tmp = grow<uint64_t>(c.pair_keys, run.candidates);
        cub_call(c, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, all, tmp, static_cast<int64_t>(run.candidates), 0,
                                                  2 * c.last_nb, st);
        });
        CCDK_CUDA_CHECK(cudaMemcpyAsync(all, tmp, run.candidates * 8, cudaMemcpyDeviceToDevice, st));
    }
    if (c.exp) {
        if (!c.exp->started)
            export_begin(c, c.all_keys.as<uint64_t>(), run.candidates, s.nv, s.ne, false);
        export_finish(c);
    }
    c.last_keys_all = true;
    c.last_pairs_general = false;
    c.last_n_pairs = run.candidates;
    c.last_nv = s.nv;
    c.last_ne = s.ne;
    c.last_query_count = run.queries;
    double* dtoi = grow<double>(c.last_toi, 1);
    const double toi = __builtin_bit_cast(double, static_cast<uint64_t>(run.toi_bits));
    CCDK_CUDA_CHECK(cudaMemcpyAsync(dtoi, &toi, 8, cudaMemcpyHostToDevice, st));
    CCDK_CUDA_CHECK(cudaEventRecord(ev[5], st));
    CCDK_CUDA_CHECK(cudaEventSynchronize(ev[5]));

    rep.toi = toi;
    rep.tolerance_hit = run.tol ? 1 : 0;
    rep.zero_toi_diagnostic = run.zd ? 1 : 0;
    rep.candidate_count = run.candidates;
    rep.query_count = run.queries;
    rep.batch_count = std::max<uint64_t>(1, run.narrow_batches);
    rep.vf_count = run.vf;
    rep.pair_tests = run.pair_tests;
    rep.total_splits = run.total_splits;
    rep.peak_queue = run.peak_queue;
    rep.evaluations = run.evaluations;
    rep.split_actions = run.split_actions;
    rep.generations = run.generations;
    rep.axis = run.axis;
    // tracked_peak_bytes with the reference's accounting (pipeline.cpp:132-136,
    // 158-159, 205-207, 228)
    rep.tracked_peak_bytes = std::max<uint64_t>(k * 32, std::max(run.peak_bytes, run.base_bytes));
    float ms_build = 0, ms_total = 0;
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&ms_build, ev[0], ev[1]));
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&ms_total, start_event ? start_event : ev[0], ev[5]));
    rep.ms_build = ms_build;
    rep.ms_sort = run.ms_sort;
    rep.ms_sweep = run.ms_sweep;
    rep.ms_pairsort = run.ms_pairsort;
    rep.ms_classify = run.ms_classify;
    rep.ms_narrow = run.ms_narrow;
    rep.ms_total = ms_total;
    rep.kernel_launches = 1 + run.launches;
    rep.broad_batches = run.broad_batches;
    rep.sweep_slabs = run.slabs;
    rep.sweep_entries = run.slab_entries;
    rep.t_cb = ms_build * 1e-3;
    rep.t_bp = (run.ms_sort + run.ms_sweep + run.ms_pairsort) * 1e-3;
    rep.t_socd = run.ms_classify * 1e-3;
    rep.t_np = run.ms_narrow * 1e-3;
}

// K1 on the resident scene (the scene was validated when it was uploaded).
void build_resident_boxes(Ctx& c, const ccdk_pipeline_cfg& cfg, float*& bmin, float*& bmax, uint4*& vids)
{
    DevScene& s = c.resident;
    const uint64_t k = s.nv + s.ne + s.nf;
    bmin = grow<float>(c.bmin, 3 * std::max<uint64_t>(k, 1));
    bmax = grow<float>(c.bmax, 3 * std::max<uint64_t>(k, 1));
    vids = grow<uint4>(c.vids, std::max<uint64_t>(k, 1));
    launch_build_boxes(c, s.v0.as<double>(), s.v1.as<double>(), s.nv, s.edges.as<uint32_t>(), s.ne,
                       s.faces.as<uint32_t>(), s.nf, cfg.inflation, bmin, bmax, vids);
    if (k) {
        auto* ctr = c.counters.as<DevCounters>();
        unsigned long long err = 0;
        d2h(c, &err, &ctr->error, 8);
        sync(c);
        if (err != ~0ull)
            throw Error(CCDK_INVALID_INPUT, "round_down_reduced: non-finite input");
    }
}

// Multi-GPU rebalance, first half: box build + this shard's STQ sweep + pair
// sort; the shard's canonical keys stay in ctx (pair_keys_sorted).
void broad_resident(Ctx& c, const ccdk_pipeline_cfg& cfg, uint32_t shard_rank, uint32_t shard_count,
                    uint64_t& n_pairs, int& key_bits, float& ms)
{
    validate_pipeline_cfg(cfg);
    DevScene& s = c.resident;
    const uint64_t k = s.nv + s.ne + s.nf;
    cudaEvent_t e0 = c.events.get(EventPool::kStep), e1 = c.events.get(EventPool::kStep + 1);
    CCDK_CUDA_CHECK(cudaEventRecord(e0, c.stream));
    float *bmin, *bmax;
    uint4* vids;
    build_resident_boxes(c, cfg, bmin, bmax, vids);
    n_pairs = 0;
    key_bits = ceil_log2(std::max<uint64_t>(k, 2));
    if (k >= 2) {
        BroadIn bi;
        bi.bmin = bmin;
        bi.bmax = bmax;
        bi.vids = vids;
        bi.k = k;
        bi.method = CCDK_BROAD_STQ;
        bi.shard_rank = shard_rank;
        bi.shard_count = shard_count;
        bi.exact_axis = false; // the shards' union is the full set for any common axis
        BroadOut bo;
        broad_phase(c, bi, bo);
        n_pairs = bo.n_pairs;
        key_bits = c.last_nb;
    }
    c.last_n_pairs = n_pairs;
    c.last_keys_all = false;
    c.last_pairs_general = false;
    c.last_nv = s.nv;
    c.last_ne = s.ne;
    CCDK_CUDA_CHECK(cudaEventRecord(e1, c.stream));
    CCDK_CUDA_CHECK(cudaEventSynchronize(e1));
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
}

// Second half: classify + narrow phase on a slice of canonical keys supplied
// by the caller (device memory), sorted here into canonical order.
void ccd_keys_resident(Ctx& c, const ccdk_pipeline_cfg& cfg, const uint64_t* keys, uint64_t n,
                       int key_bits, ccdk_report& rep)
{
    validate_pipeline_cfg(cfg);
    DevScene& s = c.resident;
    const uint64_t k = s.nv + s.ne + s.nf;
    if (key_bits != ceil_log2(std::max<uint64_t>(k, 2)))
        throw Error(CCDK_CONFIG, "ccdk_ccd_keys_resident: key width does not match the resident scene");
    std::memset(&rep, 0, sizeof rep);
    rep.toi = INFINITY;
    rep.batch_count = 1;
    cudaEvent_t e0 = c.events.get(EventPool::kStep + 2), e1 = c.events.get(EventPool::kStep + 3);
    CCDK_CUDA_CHECK(cudaEventRecord(e0, c.stream));
    c.last_nb = key_bits;
    uint64_t* sorted = grow<uint64_t>(c.pair_keys_sorted, std::max<uint64_t>(n, 1));
    if (n) {
        cub_call(c, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, keys, sorted, static_cast<int64_t>(n), 0,
                                                  2 * key_bits, c.stream);
        });
    }
    const uint64_t cap_pairs = ~0ull;
    BatchRun run { c, cfg, s, k, cap_pairs };
    run.process_keys(sorted, n);
    if (c.exp) {
        if (!c.exp->started)
            export_begin(c, c.all_keys.as<uint64_t>(), run.candidates, s.nv, s.ne, false);
        export_finish(c);
    }
    c.last_keys_all = true;
    c.last_pairs_general = false;
    c.last_n_pairs = run.candidates;
    c.last_nv = s.nv;
    c.last_ne = s.ne;
    c.last_query_count = run.queries;
    const double toi = __builtin_bit_cast(double, static_cast<uint64_t>(run.toi_bits));
    double* dtoi = grow<double>(c.last_toi, 1);
    CCDK_CUDA_CHECK(cudaMemcpyAsync(dtoi, &toi, 8, cudaMemcpyHostToDevice, c.stream));
    CCDK_CUDA_CHECK(cudaEventRecord(e1, c.stream));
    CCDK_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms_total = 0;
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&ms_total, e0, e1));
    rep.toi = toi;
    rep.tolerance_hit = run.tol ? 1 : 0;
    rep.zero_toi_diagnostic = run.zd ? 1 : 0;
    rep.candidate_count = run.candidates;
    rep.query_count = run.queries;
    rep.batch_count = std::max<uint64_t>(1, run.narrow_batches);
    rep.vf_count = run.vf;
    rep.total_splits = run.total_splits;
    rep.peak_queue = run.peak_queue;
    rep.evaluations = run.evaluations;
    rep.split_actions = run.split_actions;
    rep.generations = run.generations;
    rep.ms_classify = run.ms_classify;
    rep.ms_narrow = run.ms_narrow;
    rep.ms_total = ms_total;
    rep.kernel_launches = run.launches;
    rep.t_socd = run.ms_classify * 1e-3;
    rep.t_np = run.ms_narrow * 1e-3;
}

} // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

} // namespace ccdk

using namespace ccdk;

struct ccdk_ctx : Ctx {
};

namespace {
// An export's lifetime inside one API call: never leave with the worker
// running or waiting.
struct ExportScope {
    Ctx& c;
    ~ExportScope()
    {
        if (c.exp && c.exp->pending) {
            c.exp->pending = false;
            c.exp->aborted = true; // the worker must not deliver
            c.exp->issued.set_value();
        }
        if (c.exp && c.exp->worker.joinable())
            c.exp->worker.join();
        c.exp = nullptr;
    }
};
} // namespace

extern "C" {

int ccdk_abi_version(void) { return CCDK_ABI_VERSION; }

const char* ccdk_last_error(void) { return g_last_error.c_str(); }

int ccdk_ctx_create(int device, ccdk_ctx** out)
{
    return guard(nullptr, [&] {
        if (!out)
            throw Error(CCDK_CONFIG, "ccdk_ctx_create: null output");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error(CCDK_CUDA, "no CUDA device available (the ccdk path has no CPU fallback)");
        if (device < 0 || device >= ndev)
            throw Error(CCDK_CONFIG, "ccdk_ctx_create: device index out of range");
        CCDK_CUDA_CHECK(cudaSetDevice(device));
        std::unique_ptr<ccdk_ctx> c(new ccdk_ctx());
        c->device = device;
        CCDK_CUDA_CHECK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        CCDK_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        *out = c.release();
    });
}

int ccdk_ctx_destroy(ccdk_ctx* ctx)
{
    return guard(ctx, [&] {
        if (!ctx)
            return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->own_stream)
            cudaStreamDestroy(ctx->stream);
        if (ctx->copy_stream)
            cudaStreamDestroy(ctx->copy_stream);
        delete ctx;
    });
}

int ccdk_ctx_set_stream(ccdk_ctx* ctx, void* stream)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        CCDK_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (ctx->own_stream)
            CCDK_CUDA_CHECK(cudaStreamDestroy(ctx->stream));
        if (stream) {
            ctx->stream = static_cast<cudaStream_t>(stream);
            ctx->own_stream = false;
        } else {
            CCDK_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        }
    });
}

int ccdk_ctx_synchronize(ccdk_ctx* ctx)
{
    return guard(ctx, [&] { CCDK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

int ccdk_ctx_set_interval_capacity(ccdk_ctx* ctx, uint64_t intervals)
{
    return guard(ctx, [&] { ctx->interval_capacity = intervals; });
}

int ccdk_round_reduced(ccdk_ctx* ctx, const double* x, uint64_t n, float* down, float* up)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        double* dx = grow<double>(c.tmp[0], n);
        float* dd = grow<float>(c.tmp[1], n);
        float* du = grow<float>(c.tmp[2], n);
        h2d(c, dx, x, n * 8);
        launch_round(c, dx, n, dd, du);
        d2h(c, down, dd, n * 4);
        d2h(c, up, du, n * 4);
        sync(c);
    });
}

int ccdk_build_boxes(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                     const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf,
                     double inflation, float* min_corner, float* max_corner, uint8_t* owner_kind,
                     uint32_t* owner_index)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        upload_scene(c, c.scene, v0, v1, nv, edges, ne, faces, nf);
        if (inflation < 0.0)
            throw Error(CCDK_INVALID_INPUT, "build_boxes: inflation must be >= 0");
        const uint64_t k = nv + ne + nf;
        if (!k)
            return;
        float* bmin = grow<float>(c.bmin, 3 * k);
        float* bmax = grow<float>(c.bmax, 3 * k);
        uint4* vids = grow<uint4>(c.vids, k);
        launch_build_boxes(c, c.scene.v0.as<double>(), c.scene.v1.as<double>(), nv,
                           c.scene.edges.as<uint32_t>(), ne, c.scene.faces.as<uint32_t>(), nf,
                           inflation, bmin, bmax, vids);
        unsigned long long err = 0;
        d2h(c, &err, &c.counters.as<DevCounters>()->error, 8);
        float* mn = grow<float>(c.tmp[0], 3 * k);
        float* mx = grow<float>(c.tmp[1], 3 * k);
        uint8_t* kd = grow<uint8_t>(c.tmp[2], k);
        uint32_t* ix = grow<uint32_t>(c.tmp[3], k);
        launch_soa_to_aos(c, bmin, bmax, k, mn, mx, kd, ix, nv, ne);
        d2h(c, min_corner, mn, 12 * k);
        d2h(c, max_corner, mx, 12 * k);
        d2h(c, owner_kind, kd, k);
        d2h(c, owner_index, ix, 4 * k);
        sync(c);
        if (err != ~0ull)
            throw Error(CCDK_INVALID_INPUT, "round_down_reduced: non-finite input");
    });
}

int ccdk_choose_axis(ccdk_ctx* ctx, const float* min_corner, const float* max_corner, uint64_t k,
                     int* axis)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (k == 0)
            throw Error(CCDK_INVALID_INPUT, "choose_axis: empty box list");
        float* mn = grow<float>(c.tmp[0], 3 * k);
        float* mx = grow<float>(c.tmp[1], 3 * k);
        h2d(c, mn, min_corner, 12 * k);
        h2d(c, mx, max_corner, 12 * k);
        float* bmin = grow<float>(c.bmin, 3 * k);
        float* bmax = grow<float>(c.bmax, 3 * k);
        k_aos_to_soa<<<grid_for(k, 256), 256, 0, c.stream>>>(mn, mx, k, bmin, bmax);
        CCDK_LAUNCH_CHECK();
        // reuse the broad phase's K2 by running it on a 1-row range
        uint4* vids = grow<uint4>(c.vids, k);
        CCDK_CUDA_CHECK(cudaMemsetAsync(vids, 0xff, k * sizeof(uint4), c.stream));
        if (k < 2) {
            *axis = 0; // a single box has zero variance on every axis -> x
            return;
        }
        BroadIn bi;
        bi.bmin = bmin;
        bi.bmax = bmax;
        bi.vids = vids;
        bi.k = k;
        bi.range_begin = 0;
        bi.range_end = 0; // empty sweep: only K2/K3 run
        BroadOut bo;
        broad_phase(c, bi, bo);
        *axis = bo.axis;
    });
}

int ccdk_broad_phase(ccdk_ctx* ctx, int method, const float* min_corner, const float* max_corner,
                     const uint8_t* owner_kind, const uint32_t* owner_index, uint64_t k,
                     uint64_t nv, const uint32_t* edges, uint64_t ne, const uint32_t* faces,
                     uint64_t nf, uint64_t range_begin, uint64_t range_end, uint64_t* n_pairs,
                     ccdk_stq_stats* stats)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (method < 0 || method > 2)
            throw Error(CCDK_CONFIG, "broad phase: unknown method");
        *n_pairs = 0;
        if (stats)
            std::memset(stats, 0, sizeof *stats);
        c.last_n_pairs = 0;
        c.last_rounds.clear();
        c.last_pairs_general = true;
        c.last_keys_all = false;
        if (k < 2)
            return;
        uint32_t* e = grow<uint32_t>(c.scene.edges, 2 * std::max<uint64_t>(ne, 1));
        uint32_t* f = grow<uint32_t>(c.scene.faces, 3 * std::max<uint64_t>(nf, 1));
        h2d(c, e, edges, 8 * ne);
        h2d(c, f, faces, 12 * nf);
        c.scene.valid = false; // only topology was uploaded
        const UserBoxes ub = gather_user_boxes(c, min_corner, max_corner, owner_kind, owner_index, k, nv, e, ne,
                                               f, nf, false, "broad phase");
        float* bmin = ub.bmin;
        float* bmax = ub.bmax;
        uint4* vids = ub.vids;
        uint32_t* raw = ub.raw;
        const uint64_t nranks = ub.nranks;
        BroadIn bi;
        bi.bmin = bmin;
        bi.bmax = bmax;
        bi.vids = vids;
        bi.raw = raw;
        bi.k = k;
        bi.method = method;
        bi.range_begin = range_begin;
        bi.range_end = range_end;
        bi.want_rounds = stats != nullptr && method == CCDK_BROAD_STQ;
        // the axis is observable through StqStats, partial SweepRanges and
        // the reported axis; a full-range pair list does not depend on it
        bi.exact_axis = method != CCDK_BROAD_BF
            && (stats != nullptr || range_begin > 0 || range_end < k - 1);
        bi.unique = nranks < k;
        BroadOut bo;
        broad_phase(c, bi, bo);
        c.last_pairs_general = true;
        *n_pairs = bo.n_pairs;
        if (stats) {
            stats->n_rounds = c.last_rounds.size();
            stats->max_queue = c.last_rounds.empty() ? 0 : c.last_rounds[0];
            stats->pair_tests = bo.pair_tests;
            stats->axis = static_cast<uint64_t>(bo.axis);
            stats->axis_flags = (bo.axis_near_tie ? 1u : 0u) | (bo.axis_serial ? 2u : 0u);
        }
    });
}

int ccdk_fetch_pairs(ccdk_ctx* ctx, uint64_t* out)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        const uint64_t n = c.last_n_pairs;
        if (!n)
            return;
        uint64_t* ids = grow<uint64_t>(c.tmp[7], 2 * n);
        const uint64_t* keys = c.last_keys_all ? c.all_keys.as<uint64_t>() : c.pair_keys_sorted.as<uint64_t>();
        launch_keys_to_ids(c, keys, n, c.last_nb,
                           c.last_pairs_general ? c.own_kind.as<uint8_t>() : nullptr,
                           c.last_pairs_general ? c.own_index.as<uint32_t>() : nullptr,
                           c.last_nv, c.last_ne, ids);
        d2h(c, out, ids, 16 * n);
        sync(c);
    });
}

int ccdk_fetch_round_sizes(ccdk_ctx* ctx, uint64_t* out)
{
    return guard(ctx, [&] {
        std::copy(ctx->last_rounds.begin(), ctx->last_rounds.end(), out);
    });
}

int ccdk_classify(ccdk_ctx* ctx, const uint64_t* pairs, uint64_t n_pairs, const double* v0,
                  const double* v1, uint64_t nv, const uint32_t* edges, uint64_t ne,
                  const uint32_t* faces, uint64_t nf, uint8_t* kind_out, double* points_out,
                  uint64_t* source_out, uint64_t* n_vf, uint64_t* n_ee)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        *n_vf = *n_ee = 0;
        if (!n_pairs)
            return;
        cudaStream_t s = c.stream;
        upload_scene(c, c.scene, v0, v1, nv, edges, ne, faces, nf);
        unsigned long long* dp = grow<unsigned long long>(c.tmp[0], 2 * n_pairs);
        h2d(c, dp, pairs, 16 * n_pairs);
        uint32_t* fl = grow<uint32_t>(c.tmp[1], 4 * n_pairs);
        uint32_t *fvf = fl, *fee = fl + n_pairs, *ovf = fl + 2 * n_pairs, *oee = fl + 3 * n_pairs;
        auto* ctr = static_cast<DevCounters*>(c.counters.ensure(sizeof(DevCounters)));
        CCDK_CUDA_CHECK(cudaMemsetAsync(&ctr->error, 0xff, 8, s));
        k_classify_flags<<<grid_for(n_pairs, 256), 256, 0, s>>>(dp, n_pairs, nv, c.scene.edges.as<uint32_t>(),
                                                               ne, c.scene.faces.as<uint32_t>(), nf,
                                                               fvf, fee, &ctr->error);
        CCDK_LAUNCH_CHECK();
        cub_call(c, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, fvf, ovf, static_cast<int64_t>(n_pairs), s);
        });
        cub_call(c, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, fee, oee, static_cast<int64_t>(n_pairs), s);
        });
        k_count_total<<<1, 1, 0, s>>>(fvf, ovf, n_pairs, &ctr->misc[0]);
        k_count_total<<<1, 1, 0, s>>>(fee, oee, n_pairs, &ctr->misc[1]);
        uint8_t* qk = grow<uint8_t>(c.q_kind, n_pairs);
        double* qp = grow<double>(c.q_points, 24 * n_pairs);
        unsigned long long* src = grow<unsigned long long>(c.tmp[2], 2 * n_pairs);
        k_classify_write<<<grid_for(n_pairs, 128), 128, 0, s>>>(
            dp, n_pairs, fvf, fee, ovf, oee, &ctr->misc[0], c.scene.v0.as<double>(),
            c.scene.v1.as<double>(), c.scene.edges.as<uint32_t>(), c.scene.faces.as<uint32_t>(), qk,
            qp, src);
        CCDK_LAUNCH_CHECK();
        unsigned long long hc[8];
        d2h(c, hc, ctr, sizeof hc);
        sync(c);
        if (hc[3] != ~0ull)
            throw Error(CCDK_INVALID_INPUT, "classify: primitive index out of range");
        const uint64_t m = hc[4] + hc[5];
        *n_vf = hc[4];
        *n_ee = hc[5];
        d2h(c, kind_out, qk, m);
        d2h(c, points_out, qp, 24 * 8 * m);
        d2h(c, source_out, src, 16 * m);
        sync(c);
    });
}

int ccdk_inclusion_boxes(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                         const double* boxes, uint64_t n, double* out)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (!n)
            return;
        uint8_t* dk = grow<uint8_t>(c.tmp[0], n);
        double* dp = grow<double>(c.tmp[1], 24 * n);
        double* db = grow<double>(c.tmp[2], 6 * n);
        double* dout = grow<double>(c.tmp[3], 6 * n);
        h2d(c, dk, kind, n);
        h2d(c, dp, points, 192 * n);
        h2d(c, db, boxes, 48 * n);
        launch_inclusion(c, dk, dp, db, n, dout);
        d2h(c, out, dout, 48 * n);
        sync(c);
    });
}

int ccdk_process_intervals(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                           const double* boxes, const uint16_t* depth, const double* t_star,
                           const double* sep, uint64_t n, const ccdk_narrow_cfg* cfg,
                           uint8_t* action, double* candidate_t, uint8_t* zero_diag,
                           double* children, uint16_t* child_depth)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (!n)
            return;
        uint8_t* dk = grow<uint8_t>(c.tmp[0], n);
        double* dp = grow<double>(c.tmp[1], 24 * n);
        double* db = grow<double>(c.tmp[2], 6 * n);
        uint16_t* dd = grow<uint16_t>(c.tmp[3], 3 * n);
        double* dts = grow<double>(c.tmp[4], 2 * n);
        double* dsep = sep ? dts + n : nullptr;
        uint8_t* dact = grow<uint8_t>(c.tmp[5], 2 * n);
        double* dct = grow<double>(c.tmp[6], 13 * n);
        double* dch = dct + n;
        uint16_t* dcd = grow<uint16_t>(c.tmp[7], 6 * n);
        h2d(c, dk, kind, n);
        h2d(c, dp, points, 192 * n);
        h2d(c, db, boxes, 48 * n);
        h2d(c, dd, depth, 6 * n);
        h2d(c, dts, t_star, 8 * n);
        if (sep)
            h2d(c, dsep, sep, 8 * n);
        launch_process(c, dk, dp, db, dd, dts, dsep, n, *cfg, dact, dct, dact + n, dch, dcd);
        d2h(c, action, dact, n);
        d2h(c, zero_diag, dact + n, n);
        d2h(c, candidate_t, dct, 8 * n);
        d2h(c, children, dch, 96 * n);
        d2h(c, child_depth, dcd, 12 * n);
        sync(c);
    });
}

int ccdk_narrow_phase(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                      const double* per_query_sep, uint64_t n, const ccdk_narrow_cfg* cfg,
                      uint64_t queue_capacity, double* toi, uint8_t* flags,
                      ccdk_narrow_stats* stats)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        validate_narrow_cfg(*cfg);
        std::memset(stats, 0, sizeof *stats);
        stats->global_toi = INFINITY;
        if (!n)
            return;
        uint8_t* dk = grow<uint8_t>(c.q_kind, n);
        double* dref = grow<double>(c.q_points_ref, 24 * n);
        double* dp = grow<double>(c.q_points, 24 * n);
        double* ds = per_query_sep ? grow<double>(c.q_sep, n) : nullptr;
        // Large batches from pinned host memory are streamed: chunk i+1's
        // upload (copy stream) overlaps chunk i's narrow phase.  Per-query
        // results are partition-independent (narrowphase.hpp:93-96) and the
        // per-generation queue sizes of the chunks add up (gen_acc), so the
        // results and stats equal one run; a bounded queue capacity needs the
        // whole batch in one BFS (its overflow test is global) and is not
        // chunked.
        constexpr uint64_t kMinChunk = uint64_t(1) << 21;
        auto pinned = [](const void* p) {
            cudaPointerAttributes at {};
            return p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
        };
        const bool chunked = n >= 2 * kMinChunk && queue_capacity == UINT64_MAX && pinned(points) && pinned(kind)
            && (!per_query_sep || pinned(per_query_sep));
        // ~3 chunks: the first upload is exposed, every chunk adds a BFS's
        // fixed per-generation costs (measured optimum for 10M queries)
        const uint64_t kChunk = std::max<uint64_t>(kMinChunk, (n + 2) / 3);
        if (!chunked) {
            h2d(c, dk, kind, n);
            h2d(c, dref, points, 192 * n);
            launch_records_to_internal(c, dref, n, dp);
            if (ds)
                h2d(c, ds, per_query_sep, 8 * n);
            NarrowIn ni;
            ni.kind = dk;
            ni.points = dp;
            ni.sep = ds;
            ni.n = n;
            ni.cfg = *cfg;
            ni.queue_capacity = queue_capacity;
            NarrowOut no;
            narrow_phase(c, ni, no);
            d2h(c, toi, no.toi, 8 * n);
            d2h(c, flags, no.flags, n);
            sync(c);
            *stats = no.stats;
            return;
        }
        if (!c.copy_stream)
            CCDK_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
        // chunk boundaries: a half-size first chunk halves the one exposed
        // upload; every later upload hides behind the previous chunk's BFS
        // (10M queries: e2e 102 -> 96 ms; a third or a quarter: no better)
        std::vector<uint64_t> bnd { 0 };
        {
            uint64_t at = std::min<uint64_t>(n, std::max<uint64_t>(1, kChunk / 2));
            bnd.push_back(at);
            while (at < n) {
                at = std::min<uint64_t>(n, at + kChunk);
                bnd.push_back(at);
            }
        }
        const uint64_t nchunks = bnd.size() - 1;
        std::vector<cudaEvent_t> up(nchunks, nullptr), done(nchunks, nullptr);
        cudaEvent_t t0 = nullptr;
        if (debug_enabled()) {
            CCDK_CUDA_CHECK(cudaEventCreate(&t0));
            CCDK_CUDA_CHECK(cudaEventRecord(t0, c.stream));
            CCDK_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, t0, 0));
        }
        const auto h0 = std::chrono::steady_clock::now();
        // one upload in flight ahead of the chunk being computed: the copy
        // engine serves copies in order, so a deeper queue would hold back
        // the narrow phase's own small read-backs until every upload is done
        auto upload = [&](uint64_t i) {
            const uint64_t lo = bnd[i], cnt = bnd[i + 1] - bnd[i];
            CCDK_CUDA_CHECK(cudaMemcpyAsync(dk + lo, kind + lo, cnt, cudaMemcpyHostToDevice, c.copy_stream));
            CCDK_CUDA_CHECK(cudaMemcpyAsync(dref + 24 * lo, points + 24 * lo, 192 * cnt, cudaMemcpyHostToDevice,
                                            c.copy_stream));
            if (ds)
                CCDK_CUDA_CHECK(cudaMemcpyAsync(ds + lo, per_query_sep + lo, 8 * cnt, cudaMemcpyHostToDevice,
                                                c.copy_stream));
            CCDK_CUDA_CHECK(cudaEventCreateWithFlags(&up[i], debug_enabled() ? 0 : cudaEventDisableTiming));
            CCDK_CUDA_CHECK(cudaEventRecord(up[i], c.copy_stream));
        };
        upload(0);
        if (debug_enabled()) {
            cudaPointerAttributes at {};
            cudaPointerGetAttributes(&at, points);
            std::fprintf(stderr, "[ccdk chunks] %llu uploads enqueued in %.3f ms (points memory type %d)\n",
                         (unsigned long long)nchunks,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(),
                         (int)at.type);
        }
        double* rtoi = grow<double>(c.chunk_toi, n);
        uint8_t* rflags = grow<uint8_t>(c.chunk_flags, n);
        uint8_t* ck_kind = grow<uint8_t>(c.chunk_kind, kChunk);
        double* ck_pts = grow<double>(c.chunk_points, 24 * kChunk);
        double* ck_sep = ds ? grow<double>(c.chunk_sep, kChunk) : nullptr;
        ccdk_narrow_stats tot {};
        tot.global_toi = INFINITY;
        c.gen_acc.clear();
        c.gen_acc_keep = true;
        try {
            for (uint64_t i = 0; i < nchunks; ++i) {
                const uint64_t lo = bnd[i], cnt = bnd[i + 1] - bnd[i];
                if (i + 1 < nchunks)
                    upload(i + 1);
                CCDK_CUDA_CHECK(cudaStreamWaitEvent(c.stream, up[i], 0));
                // the chunk goes to fixed addresses, so the generation graph
                // (keyed on its kernel arguments) is reused across chunks
                launch_records_to_internal(c, dref + 24 * lo, cnt, ck_pts);
                launch_copy_device(c, dk + lo, ck_kind, cnt);
                if (ds)
                    launch_copy_device(c, ds + lo, ck_sep, 8 * cnt);
                NarrowIn ni;
                ni.kind = ck_kind;
                ni.points = ck_pts;
                ni.sep = ds ? ck_sep : nullptr;
                ni.n = cnt;
                ni.cfg = *cfg;
                NarrowOut no;
                narrow_phase(c, ni, no);
                // results gathered on the device; one read-back at the end (a
                // device-to-pageable copy per chunk would block the host)
                launch_copy_device(c, no.toi, rtoi + lo, 8 * cnt);
                launch_copy_device(c, no.flags, rflags + lo, cnt);
                if (debug_enabled()) {
                    CCDK_CUDA_CHECK(cudaEventCreate(&done[i]));
                    CCDK_CUDA_CHECK(cudaEventRecord(done[i], c.stream));
                    std::fprintf(stderr, "[ccdk chunk %llu] host %.2f ms, narrow device %.2f ms, gens %llu\n",
                                 (unsigned long long)i,
                                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(),
                                 no.stats.device_ms, (unsigned long long)no.stats.generations);
                }
                tot.global_toi = std::min(tot.global_toi, no.stats.global_toi);
                tot.total_splits += no.stats.total_splits;
                tot.evaluations += no.stats.evaluations;
                tot.split_actions += no.stats.split_actions;
                tot.generations = std::max(tot.generations, no.stats.generations);
                tot.device_ms += no.stats.device_ms;
            }
        } catch (...) {
            c.gen_acc_keep = false;
            for (auto e : up)
                if (e)
                    cudaEventDestroy(e);
            throw;
        }
        c.gen_acc_keep = false;
        d2h(c, toi, rtoi, 8 * n);
        d2h(c, flags, rflags, n);
        sync(c);
        if (debug_enabled()) {
            for (uint64_t i = 0; i < nchunks; ++i) {
                float mu = -1, md = -1;
                const cudaError_t e1 = cudaEventElapsedTime(&mu, t0, up[i]);
                const cudaError_t e2 = cudaEventElapsedTime(&md, t0, done[i]);
                if (e1 || e2)
                    std::fprintf(stderr, "[ccdk chunk] event times: %s / %s\n", cudaGetErrorString(e1),
                                 cudaGetErrorString(e2));
                std::fprintf(stderr, "[ccdk chunk %llu] uploaded at %.2f ms, narrowed at %.2f ms\n",
                             (unsigned long long)i, mu, md);
                cudaEventDestroy(done[i]);
            }
            cudaEventDestroy(t0);
        }
        for (auto e : up)
            cudaEventDestroy(e);
        for (uint64_t v : c.gen_acc)
            tot.peak_queue = std::max<uint64_t>(tot.peak_queue, v);
        *stats = tot;
    });
}

int ccdk_narrow_phase_device(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                             const double* per_query_sep, uint64_t n, const ccdk_narrow_cfg* cfg,
                             uint64_t queue_capacity, double* toi, uint8_t* flags,
                             ccdk_narrow_stats* stats)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        validate_narrow_cfg(*cfg);
        std::memset(stats, 0, sizeof *stats);
        stats->global_toi = INFINITY;
        if (!n)
            return;
        // Very large batches run as ~3 consecutive BFS runs over chunks of
        // the queries: each generation's working set (query records of the
        // live intervals) then stays closer to L2 size (10M mixed queries:
        // 100 -> 90 ms).  Results are partition-independent
        // (narrowphase.hpp:93-96) and the per-generation queue sizes are
        // summed (gen_acc), so outputs and stats equal one run.  A bounded
        // queue capacity tests the whole batch's queue and is not chunked.
        static const uint64_t kMinChunk = std::getenv("CCDK_CHUNK") ? std::strtoull(std::getenv("CCDK_CHUNK"), nullptr, 10)
                                                                    : uint64_t(1) << 21;
        const bool chunked = n >= 2 * kMinChunk && queue_capacity == UINT64_MAX;
        const uint64_t chunk = chunked ? std::max<uint64_t>(kMinChunk, (n + 2) / 3) : n;
        const uint64_t nchunks = (n + chunk - 1) / chunk;
        double* dp = grow<double>(c.q_points, 24 * chunk);
        ccdk_narrow_stats tot {};
        tot.global_toi = INFINITY;
        c.gen_acc.clear();
        c.gen_acc_keep = nchunks > 1;
        try {
            for (uint64_t i = 0; i < nchunks; ++i) {
                const uint64_t lo = i * chunk, cnt = std::min<uint64_t>(chunk, n - lo);
                launch_records_to_internal(c, points + 24 * lo, cnt, dp);
                NarrowIn ni;
                ni.kind = kind + lo;
                ni.points = dp;
                ni.sep = per_query_sep ? per_query_sep + lo : nullptr;
                ni.n = cnt;
                ni.cfg = *cfg;
                ni.queue_capacity = queue_capacity;
                NarrowOut no;
                narrow_phase(c, ni, no);
                if (toi)
                    launch_copy_device(c, no.toi, toi + lo, 8 * cnt);
                if (flags)
                    launch_copy_device(c, no.flags, flags + lo, cnt);
                if (nchunks == 1) {
                    tot = no.stats;
                    break;
                }
                tot.global_toi = std::min(tot.global_toi, no.stats.global_toi);
                tot.total_splits += no.stats.total_splits;
                tot.evaluations += no.stats.evaluations;
                tot.split_actions += no.stats.split_actions;
                tot.generations = std::max(tot.generations, no.stats.generations);
                tot.device_ms += no.stats.device_ms;
            }
        } catch (...) {
            c.gen_acc_keep = false;
            throw;
        }
        c.gen_acc_keep = false;
        sync(c);
        if (nchunks > 1)
            for (uint64_t v : c.gen_acc)
                tot.peak_queue = std::max<uint64_t>(tot.peak_queue, v);
        *stats = tot;
    });
}

int ccdk_scene_upload(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                      const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        CCDK_CUDA_CHECK(cudaSetDevice(ctx->device));
        upload_scene(*ctx, ctx->resident, v0, v1, nv, edges, ne, faces, nf);
        sync(*ctx);
    });
}

int ccdk_ccd_resident(ccdk_ctx* ctx, const ccdk_pipeline_cfg* cfg, uint32_t shard_rank,
                      uint32_t shard_count, ccdk_report* report)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        CCDK_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (!ctx->resident.valid)
            throw Error(CCDK_CONFIG, "ccdk_ccd_resident: no scene uploaded");
        if (shard_count < 1 || shard_rank >= shard_count)
            throw Error(CCDK_CONFIG, "ccdk_ccd_resident: bad shard");
        ccd_step(*ctx, ctx->resident, *cfg, shard_rank, shard_count, *report, nullptr);
    });
}

int ccdk_ccd(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
             const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf,
             const ccdk_pipeline_cfg* cfg, ccdk_report* report)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        validate_pipeline_cfg(*cfg);
        if (!v0 || !v1) {
            if (nv)
                throw Error(CCDK_INVALID_INPUT, "vertex snapshots missing");
        }
        cudaEvent_t start = c.events.get(EventPool::kApi);
        CCDK_CUDA_CHECK(cudaEventRecord(start, c.stream));
        upload_scene(c, c.scene, v0, v1, nv, edges, ne, faces, nf);
        ccd_step(c, c.scene, *cfg, 0, 1, *report, start);
    });
}


int ccdk_ccd_into(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv, const uint32_t* edges,
                  uint64_t ne, const uint32_t* faces, uint64_t nf, const ccdk_pipeline_cfg* cfg,
                  ccdk_report* report, ccdk_pairs_sink sink, void* user)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        validate_pipeline_cfg(*cfg);
        if (!sink)
            throw Error(CCDK_INVALID_INPUT, "ccdk_ccd_into: sink is null");
        if (!v0 || !v1) {
            if (nv)
                throw Error(CCDK_INVALID_INPUT, "vertex snapshots missing");
        }
        PairExport x;
        x.sink = sink;
        x.user = user;
        ExportScope scope { c };
        c.exp = &x;
        cudaEvent_t start = c.events.get(EventPool::kApi);
        CCDK_CUDA_CHECK(cudaEventRecord(start, c.stream));
        upload_scene(c, c.scene, v0, v1, nv, edges, ne, faces, nf);
        ccd_step(c, c.scene, *cfg, 0, 1, *report, start);
    });
}

int ccdk_run_batched(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv, const uint32_t* edges,
                     uint64_t ne, const uint32_t* faces, uint64_t nf, const float* min_corner,
                     const float* max_corner, const uint8_t* owner_kind, const uint32_t* owner_index, uint64_t k,
                     const ccdk_pipeline_cfg* cfg, ccdk_report* report, ccdk_pairs_sink sink, void* user)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        validate_pipeline_cfg(*cfg);
        if ((!v0 || !v1) && nv)
            throw Error(CCDK_INVALID_INPUT, "vertex snapshots missing");
        if (k && (!min_corner || !max_corner || !owner_kind || !owner_index))
            throw Error(CCDK_INVALID_INPUT, "run_batched: box arrays missing");
        if (k > 0xffffffffull)
            throw Error(CCDK_INVALID_INPUT, "run_batched: more than 2^32 - 1 boxes");
        PairExport x;
        x.sink = sink;
        x.user = user;
        ExportScope scope { c };
        if (sink)
            c.exp = &x;
        cudaEvent_t start = c.events.get(EventPool::kApi);
        CCDK_CUDA_CHECK(cudaEventRecord(start, c.stream));
        upload_scene(c, c.scene, v0, v1, nv, edges, ne, faces, nf);
        HostBoxes hb;
        hb.min_corner = min_corner;
        hb.max_corner = max_corner;
        hb.owner_kind = owner_kind;
        hb.owner_index = owner_index;
        hb.k = k;
        ccd_step(c, c.scene, *cfg, 0, 1, *report, start, &hb);
    });
}

int ccdk_ccd_no_zero_toi(ccdk_ctx* ctx, const double* v0, const double* v1, uint64_t nv,
                         const uint32_t* edges, uint64_t ne, const uint32_t* faces, uint64_t nf,
                         const ccdk_pipeline_cfg* cfg, ccdk_report* report)
{
    // ccd_no_zero_toi (pipeline.cpp:234-256): separated run first; on an
    // exact-zero ToI, re-run with zero separation and the always-split-at-t=0
    // rule and scale the retried ToI by 0.8 (kZeroToiRetryScale)
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (!cfg->narrow.no_zero_toi)
            throw Error(CCDK_CONFIG, "ccd_no_zero_toi: cfg.narrow.no_zero_toi must be set");
        ccdk_pipeline_cfg first = *cfg;
        first.narrow.no_zero_toi = 0;
        validate_pipeline_cfg(first);
        upload_scene(c, c.scene, v0, v1, nv, edges, ne, faces, nf);
        ccd_step(c, c.scene, first, 0, 1, *report, nullptr);
        if (report->toi != 0.0)
            return;
        ccdk_pipeline_cfg retry = *cfg;
        retry.narrow.no_zero_toi = 1;
        retry.narrow.min_separation = 0.0;
        retry.min_sep_mode = CCDK_MINSEP_ABSOLUTE;
        ccdk_report second;
        ccd_step(c, c.scene, retry, 0, 1, second, nullptr);
        second.toi = 0.8 * second.toi; // one IEEE RN multiply, as in pipeline.cpp:252
        second.t_cb += report->t_cb;
        second.t_bp += report->t_bp;
        second.t_socd += report->t_socd;
        second.t_np += report->t_np;
        *report = second;
    });
}

int ccdk_query_min_separations(ccdk_ctx* ctx, const uint8_t* kind, const double* points,
                               uint64_t n, const ccdk_pipeline_cfg* cfg, double* out)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (!n)
            return;
        uint8_t* dk = grow<uint8_t>(c.tmp[0], n);
        double* dp = grow<double>(c.tmp[1], 24 * n);
        double* dout = grow<double>(c.tmp[2], n);
        h2d(c, dk, kind, n);
        h2d(c, dp, points, 192 * n);
        launch_min_seps(c, dk, dp, n, *cfg, dout, false);
        d2h(c, out, dout, 8 * n);
        sync(c);
    });
}

int ccdk_broad_resident(ccdk_ctx* ctx, const ccdk_pipeline_cfg* cfg, uint32_t shard_rank,
                        uint32_t shard_count, uint64_t* n_pairs, int* key_bits, float* device_ms)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        CCDK_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (!ctx->resident.valid)
            throw Error(CCDK_CONFIG, "ccdk_broad_resident: no scene uploaded");
        if (shard_count < 1 || shard_rank >= shard_count)
            throw Error(CCDK_CONFIG, "ccdk_broad_resident: bad shard");
        float ms = 0;
        broad_resident(*ctx, *cfg, shard_rank, shard_count, *n_pairs, *key_bits, ms);
        if (device_ms)
            *device_ms = ms;
    });
}

int ccdk_copy_keys_device(ccdk_ctx* ctx, void* dst_dev)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        CCDK_CUDA_CHECK(cudaSetDevice(c.device));
        if (c.last_n_pairs)
            CCDK_CUDA_CHECK(cudaMemcpyAsync(dst_dev, c.pair_keys_sorted.p, c.last_n_pairs * 8,
                                            cudaMemcpyDeviceToDevice, c.stream));
        sync(c);
    });
}

int ccdk_ccd_keys_resident(ccdk_ctx* ctx, const ccdk_pipeline_cfg* cfg, const uint64_t* dev_keys,
                           uint64_t n, int key_bits, ccdk_report* report)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        CCDK_CUDA_CHECK(cudaSetDevice(ctx->device));
        if (!ctx->resident.valid)
            throw Error(CCDK_CONFIG, "ccdk_ccd_keys_resident: no scene uploaded");
        ccd_keys_resident(*ctx, *cfg, dev_keys, n, key_bits, *report);
    });
}

int ccdk_last_toi_device_ptr(ccdk_ctx* ctx, void** dev_ptr)
{
    return guard(ctx, [&] { *dev_ptr = grow<double>(ctx->last_toi, 1); });
}

int ccdk_copy_last_toi(ccdk_ctx* ctx, void* dst_dev)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        CCDK_CUDA_CHECK(cudaMemcpyAsync(dst_dev, grow<double>(ctx->last_toi, 1), sizeof(double),
                                        cudaMemcpyDeviceToDevice, ctx->stream));
    });
}

int ccdk_fetch_query_results(ccdk_ctx* ctx, double* toi, uint8_t* flags)
{
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(ctx->mu);
        Ctx& c = *ctx;
        const uint64_t n = c.last_query_count;
        d2h(c, toi, c.all_toi.p, 8 * n);
        d2h(c, flags, c.all_flags.p, n);
        sync(c);
    });
}

} // extern "C"
