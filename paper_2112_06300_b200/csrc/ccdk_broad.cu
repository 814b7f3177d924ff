// K2-K6: Sweep-and-Tiniest-Queue broad phase (proj/src/broadphase.cpp:12-192).
//
//   K2 choose_axis   deterministic fp64 tree reduction of centre sums and
//                    squared deviations, strict '>' argmax (broadphase.cpp:45-67)
//   K3 sort          CUB onesweep radix sort of (orderable min-key, slot):
//                    stable, -0 == +0, ties by slot = owner order
//                    (broadphase.cpp:23-35); then a gather into sorted SoA
//   K4 run ends      U[p] = first q > p with min[q] > max[p] (binary search):
//                    the STQ queue holds (p, j) in round j-p-1 for exactly the
//                    j in (p, U[p]), so StqStats follow from run lengths and a
//                    prefix sum partitions equal pair-test work per shard
//   K5 sweep         one warp per left row at a time, lanes over the row's
//                    j-window with coalesced loads of 15-bit quantised
//                    filter boxes (8 B, conservative); filter passes are
//                    compacted per warp and re-tested exactly (fp32) plus
//                    keep_pair (type + shared vertex, broadphase.cpp:12-20)
//                    32 at a time; survivors append u64 pair keys with one
//                    warp-aggregated atomic per ballot.  Windows beyond kCap
//                    spill the rest as kSeg-sized segments walked by the
//                    same code (load balance for static floors / walls
//                    whose window is ~k).
//   K6 pair sort     CUB radix sort of (lo_rank << nb | hi_rank) over 2*nb bits
//                    = canonical CandidatePair order (finalize, 37-41).
#include <math_constants.h>

#include <cub/cub.cuh>

#include "ccdk_internal.cuh"

namespace ccdk {

namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kCap = 4096; // per-row window handled by k_sweep_rows; the rest goes to k_sweep_heavy
constexpr uint32_t kSeg = 2048; // heavy-row segment length
constexpr int kRedBlocks = 256;
constexpr int kRedThreads = 256;

// ------------------------------------------------------------------- K2

__device__ __forceinline__ double centre(const float* bmin, const float* bmax, unsigned long long k,
                                         int c, unsigned long long s)
{
    return __ddiv_rn(__dadd_rn(static_cast<double>(bmin[c * k + s]),
                               static_cast<double>(bmax[c * k + s])),
                     2.0);
}

// Fixed-shape deterministic block reduction of 3 doubles.
__device__ void block_sum3(double v[3], double* out)
{
    __shared__ double sh[3][kRedThreads];
    for (int c = 0; c < 3; ++c)
        sh[c][threadIdx.x] = v[c];
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 3; ++c)
                sh[c][threadIdx.x] = __dadd_rn(sh[c][threadIdx.x], sh[c][threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 3; ++c)
            out[c] = sh[c][0];
}

__device__ void mean_from_partials(const double* part, unsigned long long k, double mean[3])
{
    double v[3] = { 0, 0, 0 };
    for (int b = threadIdx.x; b < kRedBlocks; b += kRedThreads)
        for (int c = 0; c < 3; ++c)
            v[c] = __dadd_rn(v[c], part[3 * b + c]);
    __shared__ double m[3];
    block_sum3(v, m);
    __syncthreads();
    for (int c = 0; c < 3; ++c)
        mean[c] = __ddiv_rn(m[c], static_cast<double>(k));
}

__global__ void __launch_bounds__(kRedThreads) k_axis_sum(const float* bmin, const float* bmax,
                                                          unsigned long long k, double* part)
{
    double v[3] = { 0, 0, 0 }, a[3] = { 0, 0, 0 };
    for (unsigned long long s = blockIdx.x * kRedThreads + threadIdx.x; s < k;
         s += kRedBlocks * kRedThreads)
        for (int c = 0; c < 3; ++c) {
            const double x = centre(bmin, bmax, k, c, s);
            v[c] = __dadd_rn(v[c], x);
            a[c] = __dadd_rn(a[c], fabs(x));
        }
    block_sum3(v, part + 3 * blockIdx.x);
    __syncthreads();
    block_sum3(a, part + 6 * kRedBlocks + 3 * blockIdx.x); // sum |c| for the error bound
}

__global__ void __launch_bounds__(kRedThreads) k_axis_var(const float* bmin, const float* bmax,
                                                          unsigned long long k, const double* part,
                                                          double* vpart)
{
    double mean[3];
    mean_from_partials(part, k, mean);
    double v[3] = { 0, 0, 0 };
    for (unsigned long long s = blockIdx.x * kRedThreads + threadIdx.x; s < k;
         s += kRedBlocks * kRedThreads)
        for (int c = 0; c < 3; ++c) {
            const double d = __dsub_rn(centre(bmin, bmax, k, c, s), mean[c]);
            v[c] = __dadd_rn(v[c], __dmul_rn(d, d));
        }
    __syncthreads();
    block_sum3(v, vpart + 3 * blockIdx.x);
}

// gamma_m = m u / (1 - m u), u = 2^-53 (Higham's bound for m roundings)
__device__ __forceinline__ double gamma_n(double m)
{
    const double mu = m * 0x1p-53;
    return mu / (1.0 - mu);
}

// Argmax of the tree-summed variances, and whether the reference's SERIAL
// sums (broadphase.cpp:45-67) could order the axes differently.  For either
// summation order, with n = k, A = sum |c_i| and exact mean mu:
//   |mean_hat - mu| <= dm = gamma_{n+1} A / n
//   V_hat = sum (c_i - mean_hat)^2 (1 + theta_{n+2}),
//   sum (c_i - mean_hat)^2 = V* + n (mean_hat - mu)^2     (V* exact),
// so serial and tree variances differ by at most 2 gamma_{n+2} V + 2 n dm^2
// (+ second order); R below is twice that.  If the chosen axis's interval
// [V - R, V + R] is disjoint from every other axis's, the serial argmax
// (strict '>', ties to the lower axis) is the same axis; otherwise flag
// the serial recomputation (k_axis_serial).
__global__ void __launch_bounds__(kRedThreads) k_axis_pick(const double* part, unsigned long long k,
                                                           int* axis)
{
    const double* vpart = part + 3 * kRedBlocks;
    const double* apart = part + 6 * kRedBlocks;
    double v[3] = { 0, 0, 0 }, a[3] = { 0, 0, 0 };
    for (int b = threadIdx.x; b < kRedBlocks; b += kRedThreads)
        for (int c = 0; c < 3; ++c) {
            v[c] = __dadd_rn(v[c], vpart[3 * b + c]);
            a[c] = __dadd_rn(a[c], apart[3 * b + c]);
        }
    __shared__ double var[3], abs_sum[3];
    block_sum3(v, var);
    __syncthreads();
    block_sum3(a, abs_sum);
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = 0;
        for (int c = 1; c < 3; ++c)
            if (var[c] > var[best])
                best = c;
        const double n = static_cast<double>(k);
        const double g = gamma_n(n + 3.0);
        double R[3];
        for (int c = 0; c < 3; ++c) {
            const double dm = gamma_n(n + 2.0) * abs_sum[c] * (1.0 + 4.0 * g) / n;
            R[c] = 4.0 * g * var[c] + 4.0 * n * dm * dm + 0x1p-1000;
        }
        int uncertain = 0;
        for (int c = 0; c < 3; ++c)
            if (c != best && var[best] - R[best] <= var[c] + R[c])
                uncertain = 1;
        axis[0] = best;
        axis[1] = uncertain;
    }
}

// The reference's choose_axis in its own summation order, for inputs whose
// tree-summed variances are within the error bound of a tie (regular meshes
// without jitter: symmetric extents give equal variances up to rounding).
// One warp per axis; the warp stages 1024 centres in shared memory and lane 0
// adds them in index order, so the result is bit-identical to the serial
// loop.  Runs (and costs ~2 dependent DADDs per box) only when axis[1] is set.
constexpr int kSerialChunk = 1024;
__global__ void __launch_bounds__(96) k_axis_serial(const float* bmin, const float* bmax,
                                                   unsigned long long k, int* axis)
{
    if (!axis[1])
        return;
    __shared__ double stage[3][kSerialChunk];
    __shared__ double var[3];
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* st = stage[c];
    double mean = 0.0, acc = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        acc = 0.0;
        for (unsigned long long s0 = 0; s0 < k; s0 += kSerialChunk) {
            const unsigned long long cnt = k - s0 < kSerialChunk ? k - s0 : kSerialChunk;
            for (unsigned long long i = lane; i < cnt; i += 32)
                st[i] = centre(bmin, bmax, k, c, s0 + i);
            __syncwarp();
            if (lane == 0) {
                if (pass == 0) {
                    for (unsigned long long i = 0; i < cnt; ++i)
                        acc = __dadd_rn(acc, st[i]);
                } else {
                    for (unsigned long long i = 0; i < cnt; ++i) {
                        const double d = __dsub_rn(st[i], mean);
                        acc = __dadd_rn(acc, __dmul_rn(d, d));
                    }
                }
            }
            __syncwarp();
        }
        mean = __shfl_sync(0xffffffffu, __ddiv_rn(acc, static_cast<double>(k)), 0);
    }
    if (lane == 0)
        var[c] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = 0;
        for (int a = 1; a < 3; ++a)
            if (var[a] > var[best])
                best = a;
        axis[0] = best;
        axis[2] = 1; // the serial order decided
    }
}

// ------------------------------------------------------------------- K3

__device__ __forceinline__ uint32_t orderable(float x)
{
    uint32_t u = __float_as_uint(x);
    if (u == 0x80000000u)
        u = 0; // -0 == +0 under the reference's float comparator
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void k_sort_keys(const float* bmin, unsigned long long k, const int* axis,
                            uint32_t* keys, uint32_t* vals)
{
    const unsigned long long s = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (s >= k)
        return;
    keys[s] = orderable(bmin[static_cast<unsigned long long>(*axis) * k + s]);
    vals[s] = static_cast<uint32_t>(s);
}

// ---- quantised 2-axis filter boxes for the sweep.
// The sweep's pair test on the two non-sweep axes runs first on 15-bit
// quantised boxes (8 bytes instead of 16): q = floor((x - lo) * s) for a min,
// ceil(...) for a max, clamped to [0, 32767], with the same fp32 operations
// for every box.  That map is monotone non-decreasing, so min_j <= max_i
// implies q(min_j) <= q(max_i): the quantised test passes every exactly
// overlapping pair (a superset), and each pass is re-tested on the exact
// fp32 box before keep_pair.  The sweep is L1-bandwidth bound, so halving
// the bytes per test is what matters.
__device__ __forceinline__ unsigned f2ord(float f)
{
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned o)
{
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// qb[0..2] = ordered min of bmin per axis, qb[3..5] = ordered max of bmax
// (qb pre-set to 0xffffffff / 0).
__global__ void k_quant_bounds(const float* bmin, const float* bmax, unsigned long long k, unsigned* qb)
{
    unsigned lo[3] = { 0xffffffffu, 0xffffffffu, 0xffffffffu }, hi[3] = { 0, 0, 0 };
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = min(lo[a], f2ord(bmin[a * k + i]));
            hi[a] = max(hi[a], f2ord(bmax[a * k + i]));
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&qb[a], lo[a]);
            atomicMax(&qb[3 + a], hi[a]);
        }
    }
}

struct QuantAxis {
    float lo, s;
};
__device__ __forceinline__ QuantAxis quant_axis(const unsigned* qb, int a)
{
    const float lo = ord2f(qb[a]), hi = ord2f(qb[3 + a]);
    const float ext = __fsub_rn(hi, lo);
    QuantAxis q { lo, 0.0f };
    if (isfinite(lo) && isfinite(hi) && isfinite(ext) && ext > 0.0f)
        q.s = __fdiv_rn(32767.0f, ext);
    if (!isfinite(q.s)) // denormal extent
        q.s = 0.0f;
    return q; // s == 0: every box quantises to 0 (the filter passes all)
}
__device__ __forceinline__ unsigned quant_dn(QuantAxis q, float x)
{
    const float v = floorf(__fmul_rn(__fsub_rn(x, q.lo), q.s));
    return v <= 0.0f ? 0u : v >= 32767.0f ? 32767u : static_cast<unsigned>(v);
}
__device__ __forceinline__ unsigned quant_up(QuantAxis q, float x)
{
    const float v = ceilf(__fmul_rn(__fsub_rn(x, q.lo), q.s));
    return v <= 0.0f ? 0u : v >= 32767.0f ? 32767u : static_cast<unsigned>(v);
}

__global__ void k_permute(const float* bmin, const float* bmax, const uint4* vids,
                          const uint32_t* raw, unsigned long long k, const int* axis,
                          const uint32_t* order, float* smin_a, float* smax_a, float4* sbox,
                          uint4* svid, uint32_t* sraw, const unsigned* qb, uint2* sq)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (p >= k)
        return;
    const int a = *axis, a1 = (a + 1) % 3, a2 = (a + 2) % 3;
    const unsigned long long s = order[p];
    smin_a[p] = bmin[a * k + s];
    smax_a[p] = bmax[a * k + s];
    const float4 b = make_float4(bmin[a1 * k + s], bmax[a1 * k + s], bmin[a2 * k + s], bmax[a2 * k + s]);
    sbox[p] = b;
    const QuantAxis q1 = quant_axis(qb, a1), q2 = quant_axis(qb, a2);
    // hi word stored with the guard bits set (see qhit)
    sq[p] = make_uint2(quant_dn(q1, b.x) | (quant_dn(q2, b.z) << 16),
                       quant_up(q1, b.y) | (quant_up(q2, b.w) << 16) | 0x80008000u);
    svid[p] = vids[s];
    if (sraw)
        sraw[p] = raw ? raw[s] : static_cast<uint32_t>(s);
}

// ------------------------------------------------------------------- K4

// Sum of a per-thread count over the block, one atomic per block (every thread
// of a 256-thread block must call it): a per-warp atomic on one address
// serialises ~k/32 updates at L2 (~45 us at C4's 1.5M slab entries).
constexpr int kSumBlock = 256;
__device__ __forceinline__ void block_add(unsigned long long* dst, unsigned long long v)
{
    __shared__ unsigned long long part[kSumBlock / 32];
    for (int o = 16; o; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0)
        part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < kSumBlock / 32; ++i)
            t += part[i];
        if (t)
            atomicAdd(dst, t);
    }
}

__global__ void __launch_bounds__(kSumBlock) k_run_ends(const float* smin_a, const float* smax_a, unsigned long long k,
                           unsigned long long lo, unsigned long long hi, uint32_t* run_end,
                           unsigned long long* run_len, unsigned long long* pair_tests)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    unsigned long long len = 0;
    if (p < k) {
        unsigned long long end = p + 1;
        if (p >= lo && p < hi) {
            const float reach = smax_a[p];
            unsigned long long a = p + 1, b = k;
            while (a < b) { // upper_bound of reach in smin_a[p+1, k)
                const unsigned long long m = (a + b) >> 1;
                if (smin_a[m] <= reach)
                    a = m + 1;
                else
                    b = m;
            }
            end = a;
            len = end - p - 1;
        }
        run_end[p] = static_cast<uint32_t>(end);
        if (run_len)
            run_len[p] = len;
    }
    block_add(pair_tests, len);
}

// shard boundaries: first p with exclusive prefix >= W*r/S
__global__ void k_shard_range(const unsigned long long* incl, unsigned long long lo,
                              unsigned long long hi, uint32_t rank, uint32_t count,
                              unsigned long long* range)
{
    if (threadIdx.x > 1)
        return;
    const unsigned long long W = hi > lo ? incl[hi - 1] : 0;
    const uint32_t r = rank + threadIdx.x;
    unsigned long long pos;
    if (r == 0) {
        pos = lo;
    } else if (r >= count) {
        pos = hi;
    } else {
        const unsigned long long T = (W / count) * r + ((W % count) * r) / count; // floor(W*r/S)
        // exclusive prefix E[p] = incl[p] - len(p) = incl[p-1]; find first p in
        // [lo, hi) with E[p] >= T, i.e. first p with (p == lo ? 0 : incl[p-1]) >= T
        unsigned long long a = lo, b = hi;
        while (a < b) {
            const unsigned long long m = (a + b) >> 1;
            const unsigned long long e = m == lo ? 0 : incl[m - 1];
            if (e >= T)
                b = m;
            else
                a = m + 1;
        }
        pos = a;
    }
    range[threadIdx.x] = pos;
}

__global__ void k_full_range(unsigned long long lo, unsigned long long hi, unsigned long long* range)
{
    range[0] = lo;
    range[1] = hi;
}

__global__ void k_heavy_count(const uint32_t* run_end, const unsigned long long* range,
                              unsigned long long k, uint32_t* nseg, uint32_t cap, uint32_t seg)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (p >= k)
        return;
    uint32_t n = 0;
    if (p >= range[0] && p < range[1]) {
        const unsigned long long start = p + 1 + cap;
        const unsigned long long end = run_end[p];
        if (end > start)
            n = static_cast<uint32_t>((end - start + seg - 1) / seg);
    }
    nseg[p] = n;
}

struct Seg {
    uint32_t p, jb, je, pad;
};

__global__ void k_heavy_gen(const uint32_t* run_end, const uint32_t* nseg, const uint32_t* off,
                            unsigned long long k, Seg* segs, unsigned long long* n_heavy, uint32_t cap,
                            uint32_t seg)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (p >= k)
        return;
    const uint32_t n = nseg[p];
    if (p == k - 1)
        *n_heavy = static_cast<unsigned long long>(off[p]) + n;
    if (!n)
        return;
    const uint32_t start = static_cast<uint32_t>(p + 1 + cap);
    const uint32_t end = run_end[p];
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t jb = start + i * seg;
        const uint32_t je = min(end, jb + seg);
        segs[off[p] + i] = { static_cast<uint32_t>(p), jb, je, 0 };
    }
}

// ------------------------------------------------------------------- K5

struct SweepArgs {
    const float* smin_a;
    const float* smax_a;
    const float4* sbox;
    const uint2* sq;           // quantised filter boxes (lo = qmin_b | qmin_c << 16, hi = qmax_b | qmax_c << 16)
    const uint4* svid;
    const uint32_t* sraw;      // bf mode only
    const uint32_t* run_end;
    const unsigned long long* range;
    unsigned long long row0;   // first row covered by the grid
    unsigned long long k;
    int nb;
    int bf;                    // bf: raw-position range filter + full axis test
    unsigned long long bf_lo, bf_hi;
    unsigned long long* keys;
    unsigned long long cap;
    unsigned long long* n_pairs;
    const Seg* segs;
    const unsigned long long* n_heavy;
    unsigned long long short_len; // rows with windows <= this go to k_sweep_short (0: none)
    unsigned long long row_cap;   // per-row window handled by k_sweep_rows; the rest: heavy segments
    // slab mode: entry's slab and its box's first slab; a pair is emitted only
    // in its canonical slab max(first_p, first_q)
    const uint32_t* slab;
    const uint32_t* slab_first;
};

// keep_pair (broadphase.cpp:12-20) on vertex triples: the count of present
// vertices is the primitive kind (1 V, 2 E, 3 F).
__device__ __forceinline__ bool keep_pair(uint4 a, uint4 b)
{
    const int na = 1 + (a.y != kNone) + (a.z != kNone);
    const int nb = 1 + (b.y != kNone) + (b.z != kNone);
    if (na + nb == 4) {
        if (na != 2) { // vertex-face
            const uint32_t v = na == 1 ? a.x : b.x;
            const uint4 f = na == 1 ? b : a;
            return v != f.x && v != f.y && v != f.z;
        }
        return a.x != b.x && a.x != b.y && a.y != b.x && a.y != b.y; // edge-edge
    }
    return false;
}

__device__ __forceinline__ bool box_hit(float4 m, float4 o)
{
    return o.x <= m.y && m.x <= o.y && o.z <= m.w && m.z <= o.w;
}

// Kept pairs of a warp wait in shared memory and go out 32 at a time with one
// warp-aggregated atomic.  Most quantised hits fail the exact test or
// keep_pair (neighbouring triangles share vertices; a floor face pairs only
// with vertices), so emitting per drain would pay the atomic's round trip
// for a handful of keys.
constexpr int kOutBuf = 64;
struct WarpOut {
    unsigned long long* buf; // kOutBuf keys, per warp in shared memory
    unsigned n;              // warp-uniform
};

__device__ __forceinline__ void out_flush(const SweepArgs& a, WarpOut& o, unsigned cnt, unsigned lane)
{
    unsigned long long base = 0;
    if (lane == 0)
        base = atomicAdd(a.n_pairs, static_cast<unsigned long long>(cnt));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < cnt && base + lane < a.cap)
        a.keys[base + lane] = o.buf[lane];
}

// append the lanes' kept pairs; flush whenever 32 are waiting
__device__ __forceinline__ void out_push(const SweepArgs& a, WarpOut& o, bool keep, uint32_t ra, uint32_t rb,
                                         unsigned lane)
{
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m)
        return;
    if (keep) {
        const uint32_t lo = min(ra, rb), hi = max(ra, rb);
        o.buf[o.n + __popc(m & ((1u << lane) - 1))] = (static_cast<unsigned long long>(lo) << a.nb) | hi;
    }
    o.n += __popc(m);
    __syncwarp();
    if (o.n >= 32) {
        out_flush(a, o, 32, lane);
        const unsigned rem = o.n - 32;
        const unsigned long long v = lane < rem ? o.buf[32 + lane] : 0ull;
        __syncwarp();
        if (lane < rem)
            o.buf[lane] = v;
        __syncwarp();
        o.n = rem;
    }
}

__device__ __forceinline__ void out_finish(const SweepArgs& a, WarpOut& o, unsigned lane)
{
    if (o.n)
        out_flush(a, o, o.n, lane);
    o.n = 0;
}

__device__ __forceinline__ bool bf_ok(const SweepArgs& a, unsigned long long p, unsigned long long j)
{
    if (!a.bf)
        return true;
    const uint32_t r = min(a.sraw[p], a.sraw[j]);
    return r >= a.bf_lo && r < a.bf_hi && a.smin_a[p] <= a.smax_a[j];
}

// K5 sweep, row-parallel form: one warp per row at a time, lanes over the
// row's window [p+1, min(run_end, p+1+kCap)) in 32-box strides with
// coalesced float4 loads.  A warp walks kRowsPerWarp consecutive rows and a
// CTA 8 warps of them, so neighbouring windows (which overlap almost
// entirely) are served from L1; no block barrier, and a lane tests only boxes
// of its own row's window (the ragged tail costs < 32 lanes per row).
// Three-axis overlaps (~3% of tests on cloth, so most 32-box strides hold
// one) are compacted into a per-warp list and the adjacency/kind filter
// (keep_pair, which needs the other box's vertex ids) runs on 32 of them at a
// time with every lane busy, instead of a dependent load per stride.  Rows
// whose window exceeds kCap spill the rest to k_sweep_heavy segments.
#ifndef CCDK_SWEEP_RPW
#define CCDK_SWEEP_RPW 8
#endif
#ifndef CCDK_SWEEP_TB
#define CCDK_SWEEP_TB 512
#endif
constexpr int kRowsPerWarp = CCDK_SWEEP_RPW;
constexpr int kRowsTB = CCDK_SWEEP_TB;
#ifndef CCDK_SWEEP_UNROLL
#define CCDK_SWEEP_UNROLL 4
#endif
constexpr int kUnroll = CCDK_SWEEP_UNROLL;
constexpr int kHitBuf = 32 * kUnroll + 32; // < 32 left over + kUnroll strides

__device__ __forceinline__ void filter_hits(const SweepArgs& a, unsigned long long p, float4 mb, uint4 mv,
                                            const unsigned* hits, unsigned cnt, unsigned lane, WarpOut& o)
{
    bool h = lane < cnt;
    const unsigned long long q = p + (h ? hits[lane] : 0u);
    // the quantised pass is a superset: the exact fp32 test decides; the box
    // and the vertex ids load together (one round trip)
    const float4 ob = a.sbox[q];
    const uint4 ov = a.svid[q];
    h = h && box_hit(mb, ob);
    if (a.slab) // slab mode: only the canonical slab of the pair emits it
        h = h && max(a.slab_first[p], a.slab_first[q]) == a.slab[p];
    out_push(a, o, h && keep_pair(mv, ov) && bf_ok(a, p, q), mv.w, ov.w, lane);
}

// Run the filter on every full chunk of 32 (all of them when `all`) and
// move the remainder to the front of the list.
__device__ __forceinline__ void drain_hits(const SweepArgs& a, unsigned long long p, float4 mb, uint4 mv,
                                           unsigned* hits, unsigned& nh, unsigned lane, bool all, WarpOut& o)
{
    __syncwarp();
    unsigned base = 0;
    while (nh - base >= 32 || (all && nh > base)) {
        const unsigned cnt = min(nh - base, 32u);
        filter_hits(a, p, mb, mv, hits + base, cnt, lane, o);
        base += cnt;
    }
    const unsigned rem = nh - base; // < 32
    const unsigned v = lane < rem ? hits[base + lane] : 0u;
    __syncwarp();
    if (lane < rem)
        hits[lane] = v;
    __syncwarp();
    nh = rem;
}

__device__ __forceinline__ void push_hit(unsigned* hits, unsigned& nh, bool h, unsigned off, unsigned lane)
{
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if (h)
        hits[nh + __popc(m & ((1u << lane) - 1))] = off;
    nh += __popc(m);
}

// Quantised 2-axis overlap (superset of the exact test): per 16-bit lane,
// (0x8000 + a) - b keeps bit 15 iff a >= b (15-bit values: no borrow across
// lanes), so one subtract checks both axes of one inequality.
// Both operands' hi words carry the guard bits already (set at quantisation).
constexpr unsigned kGuard = 0x80008000u;
__device__ __forceinline__ bool qhit(unsigned m_hi_g, unsigned m_lo, uint2 o)
{
    const unsigned x1 = m_hi_g - o.x; // o.qmin <= m.qmax
    const unsigned x2 = o.y - m_lo;   // m.qmin <= o.qmax
    return (x1 & x2 & kGuard) == kGuard;
}

// Row p against boxes [jb, je) of its window (warp-cooperative).
__device__ __forceinline__ void sweep_window(const SweepArgs& a, unsigned long long p, unsigned long long jb,
                                             unsigned long long je, unsigned* hits, unsigned lane, WarpOut& o)
{
    const float4 mb = a.sbox[p];
    const uint4 mv = a.svid[p];
    const uint2 mq = a.sq[p];
    const unsigned m_hi_g = mq.y, m_lo = mq.x;
    unsigned nh = 0;             // warp-uniform
    unsigned long long j0 = jb;  // warp-uniform stride base
    // kUnroll full strides per iteration: all loads in flight before the
    // tests; one advancing pointer, so the loads use immediate offsets
    const uint2* qp = a.sq + j0 + lane;
    unsigned off = static_cast<unsigned>(j0 - p) + lane; // this lane's box offset from p
    for (; j0 + 32 * kUnroll <= je; j0 += 32 * kUnroll, qp += 32 * kUnroll, off += 32 * kUnroll) {
        uint2 qv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            qv[u] = __ldg(qp + 32 * u);
        bool h[kUnroll], any = false;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            h[u] = qhit(m_hi_g, m_lo, qv[u]);
            any = any || h[u];
        }
        if (__any_sync(0xffffffffu, any)) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                push_hit(hits, nh, h[u], off + 32 * u, lane);
            if (nh >= 32)
                drain_hits(a, p, mb, mv, hits, nh, lane, false, o);
        }
    }
    // ragged tail (< 32 kUnroll boxes): lanes past the window end are idle
    for (; j0 < je; j0 += 32) {
        const unsigned long long j = j0 + lane;
        const bool valid = j < je;
        const bool h = valid && qhit(m_hi_g, m_lo, __ldg(&a.sq[valid ? j : p]));
        push_hit(hits, nh, h, static_cast<unsigned>(j - p), lane);
    }
    if (nh)
        drain_hits(a, p, mb, mv, hits, nh, lane, true, o);
}

#ifndef CCDK_SWEEP_MINB
#define CCDK_SWEEP_MINB 3
#endif
__global__ void __launch_bounds__(kRowsTB, CCDK_SWEEP_MINB) k_sweep_rows(SweepArgs a)
{
    __shared__ unsigned s_hits[kRowsTB / 32][kHitBuf];
    __shared__ unsigned long long s_out[kRowsTB / 32][kOutBuf];
    const unsigned lane = threadIdx.x & 31;
    unsigned* hits = s_hits[threadIdx.x >> 5];
    WarpOut o { s_out[threadIdx.x >> 5], 0u };
    const unsigned long long B = a.range[0], E = a.range[1];
    const unsigned long long warp = (blockIdx.x * static_cast<unsigned long long>(kRowsTB) + threadIdx.x) >> 5;
    const unsigned long long p0 = a.row0 + warp * kRowsPerWarp;
    for (int r = 0; r < kRowsPerWarp; ++r) {
        const unsigned long long p = p0 + r;
        if (p >= E)
            break; // warp-uniform
        if (p < B)
            continue;
        const unsigned long long re = a.run_end[p];
        if (re <= p + 1 + a.short_len)
            continue; // empty, or a short window (k_sweep_short)
        const unsigned long long je = min(re, p + 1 + a.row_cap);
        sweep_window(a, p, p + 1, je, hits, lane, o);
    }
    out_finish(a, o, lane);
}

// Short windows (slab mode: ~20 boxes per window, so a warp per row would
// leave most lanes idle and pay the per-row set-up 1.5M times): one LANE per
// row, the warp stepping through its 32 rows' windows in lockstep (trip count
// = the longest of them, <= short_len).  Quantised hits are compacted as
// (owner lane, other entry) into a per-warp list and the exact test,
// keep_pair and the slab dedup run on 32 of them at a time with every lane
// busy, emitted with one warp-aggregated atomic.
constexpr int kShortBuf = 64;

__device__ __forceinline__ void short_filter(const SweepArgs& a, unsigned long long p_base, const uint2* hits,
                                             unsigned cnt, unsigned lane, WarpOut& o)
{
    bool h = lane < cnt;
    const uint2 e = h ? hits[lane] : make_uint2(0, 0);
    const unsigned long long p = p_base + e.x, q = e.y;
    // every operand in one round trip (no load waits on another's test)
    const float4 mb = a.sbox[p], ob = a.sbox[q];
    const uint4 mv = a.svid[p], ov = a.svid[q];
    h = h && box_hit(mb, ob);
    if (a.slab)
        h = h && max(a.slab_first[p], a.slab_first[q]) == a.slab[p];
    out_push(a, o, h && keep_pair(mv, ov), mv.w, ov.w, lane);
}

__global__ void __launch_bounds__(kRowsTB) k_sweep_short(SweepArgs a)
{
    __shared__ uint2 s_hits[kRowsTB / 32][kShortBuf];
    __shared__ unsigned long long s_out[kRowsTB / 32][kOutBuf];
    const unsigned lane = threadIdx.x & 31;
    uint2* hits = s_hits[threadIdx.x >> 5];
    WarpOut o { s_out[threadIdx.x >> 5], 0u };
    const unsigned long long B = a.range[0], E = a.range[1];
    const unsigned long long p_base = a.row0 + ((blockIdx.x * static_cast<unsigned long long>(kRowsTB) + threadIdx.x) & ~31ull);
    if (p_base >= E)
        return; // warp-uniform
    const unsigned long long p = p_base + lane;
    unsigned len = 0;
    uint2 mq = make_uint2(0, 0);
    if (p >= B && p < E) {
        const unsigned long long re = a.run_end[p];
        if (re > p + 1 && re <= p + 1 + a.short_len) {
            len = static_cast<unsigned>(re - p - 1);
            mq = a.sq[p];
        }
    }
    const unsigned maxlen = __reduce_max_sync(0xffffffffu, len);
    const unsigned lt = (1u << lane) - 1;
    unsigned nh = 0; // warp-uniform
    for (unsigned t = 0; t < maxlen; ++t) {
        const unsigned long long q = p + 1 + t;
        const bool h = t < len && qhit(mq.y, mq.x, __ldg(&a.sq[q]));
        const unsigned m = __ballot_sync(0xffffffffu, h);
        if (h)
            hits[nh + __popc(m & lt)] = make_uint2(lane, static_cast<unsigned>(q));
        nh += __popc(m);
        if (nh >= 32) {
            __syncwarp();
            short_filter(a, p_base, hits, 32, lane, o);
            const unsigned rem = nh - 32;
            const uint2 v = lane < rem ? hits[32 + lane] : make_uint2(0, 0);
            __syncwarp();
            if (lane < rem)
                hits[lane] = v;
            __syncwarp();
            nh = rem;
        }
    }
    if (nh) {
        __syncwarp();
        short_filter(a, p_base, hits, nh, lane, o);
    }
    out_finish(a, o, lane);
}

// Heavy rows: one warp per (row, kSeg-long window segment) — the part of a
// window beyond kCap (static floors / container walls whose window is ~k).
__global__ void __launch_bounds__(kRowsTB) k_sweep_heavy(SweepArgs a)
{
    __shared__ unsigned s_hits[kRowsTB / 32][kHitBuf];
    __shared__ unsigned long long s_out[kRowsTB / 32][kOutBuf];
    const unsigned lane = threadIdx.x & 31;
    unsigned* hits = s_hits[threadIdx.x >> 5];
    WarpOut o { s_out[threadIdx.x >> 5], 0u };
    const unsigned long long nseg = *a.n_heavy;
    const unsigned long long warp = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) >> 5;
    const unsigned long long nwarps = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
    for (unsigned long long sg = warp; sg < nseg; sg += nwarps) {
        const Seg g = a.segs[sg];
        sweep_window(a, g.p, g.jb, g.je, hits, lane, o);
    }
    out_finish(a, o, lane);
}

// ---- K5' slab mode.  The candidate set is a property of the boxes alone
// (closed overlap on all three axes + keep_pair, broadphase.cpp:12-20, 69-127),
// not of the sweep that enumerates it, so any exact enumeration yields it.  A
// 1-D sweep along the max-variance axis a tests every pair whose intervals
// overlap on a: on a 410 x 410 cloth that is ~2,700 boxes per window (2.7e9
// tests at C4), 97% of which miss on another axis.  Slab mode cuts space along
// a second axis b into S slabs about twice the mean box extent wide, inserts
// each box into every slab its b-interval touches, and sweeps every slab along
// a exactly like K5: a window now holds only the boxes of one slab.  The slab
// map s(x) = clamp(floor((x - lo) * inv_w)) is the same fp32 sequence for every
// box, hence monotone, so two boxes that overlap on b both appear in slab
// max(s(min_i), s(min_j)) — the first slab of the intersection of their slab
// ranges — and the sweep emits a pair only there: exactly once.  Used for the
// full-range broad phase (ccd's default step, stq/sap/bf without StqStats or
// SweepRange); StqStats, SweepRange slices, budget halving and multi-GPU shards
// keep the 1-D sweep whose positions they are defined on.
struct SlabParams {
    float lo, inv_w;
    unsigned S;
    int side; // 0: b = (a+1)%3 (sbox.x/.y), 1: b = (a+2)%3 (sbox.z/.w)
    int ok;
};
constexpr unsigned kMaxSlabs = 65535; // slab ids sort on 16 bits
constexpr unsigned kShortLen = 64;    // slab-mode windows up to this run one lane per row
constexpr uint32_t kSlabCap = 256;    // slab mode: row cap and heavy segment length
constexpr uint64_t kSlabMinBoxes = 200000; // measured crossover (C1 75k: 1-D faster; C2 300k: slab faster)

__device__ __forceinline__ unsigned slab_of(const SlabParams& P, float x)
{
    const float f = floorf(__fmul_rn(__fsub_rn(x, P.lo), P.inv_w));
    return f <= 0.0f ? 0u : f >= static_cast<float>(P.S - 1) ? P.S - 1 : static_cast<unsigned>(f);
}

// sums of the box extents along the two non-sweep axes (sorted boxes)
__global__ void k_slab_stats(const float4* sbox, unsigned long long k, double* sums)
{
    double e1 = 0.0, e2 = 0.0;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const float4 b = sbox[i];
        e1 += static_cast<double>(b.y) - static_cast<double>(b.x);
        e2 += static_cast<double>(b.w) - static_cast<double>(b.z);
    }
    for (int o = 16; o; o >>= 1) {
        e1 += __shfl_xor_sync(0xffffffffu, e1, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sums[0], e1);
        atomicAdd(&sums[1], e2);
    }
}

// slab axis = the wider of the two non-sweep axes; width = 2 x its mean box
// extent (at least ext / kMaxSlabs); ok = finite bounds and >= 2 slabs
__global__ void k_slab_params(const unsigned* qb, const int* axis, const double* sums, unsigned long long k,
                              double width_factor, SlabParams* P)
{
    const int a = *axis, a1 = (a + 1) % 3, a2 = (a + 2) % 3;
    const float lo1 = ord2f(qb[a1]), hi1 = ord2f(qb[3 + a1]);
    const float lo2 = ord2f(qb[a2]), hi2 = ord2f(qb[3 + a2]);
    const double ext1 = static_cast<double>(hi1) - lo1, ext2 = static_cast<double>(hi2) - lo2;
    const int side = ext2 > ext1 ? 1 : 0;
    const float lo = side ? lo2 : lo1;
    const double ext = side ? ext2 : ext1;
    const double mean = sums[side] / static_cast<double>(k);
    SlabParams p { lo, 0.0f, 1u, side, 0 };
    if (isfinite(lo1) && isfinite(hi1) && isfinite(lo2) && isfinite(hi2) && ext > 0.0) {
        const double w = fmax(width_factor * mean, ext / kMaxSlabs);
        const double S = ceil(ext / w);
        if (S >= 2.0 && w > 0.0) {
            p.S = static_cast<unsigned>(fmin(S, static_cast<double>(kMaxSlabs)));
            p.inv_w = static_cast<float>(1.0 / w);
            p.ok = isfinite(p.inv_w) && p.inv_w > 0.0f;
        }
    }
    *P = p;
}

__global__ void k_slab_count(const float4* sbox, unsigned long long k, const SlabParams* Pp, uint32_t* cnt)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (p >= k)
        return;
    const SlabParams P = *Pp;
    const float4 b = sbox[p];
    const float mn = P.side ? b.z : b.x, mx = P.side ? b.w : b.y;
    cnt[p] = slab_of(P, mx) - slab_of(P, mn) + 1;
}

// entries in sorted-position order: (slab, position) for every slab a box touches
__global__ void k_slab_emit(const float4* sbox, unsigned long long k, const SlabParams* Pp, const uint32_t* off,
                            uint32_t* keys, uint32_t* vals)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (p >= k)
        return;
    const SlabParams P = *Pp;
    const float4 b = sbox[p];
    const unsigned s0 = slab_of(P, P.side ? b.z : b.x), s1 = slab_of(P, P.side ? b.w : b.y);
    uint32_t o = off[p];
    for (unsigned s = s0; s <= s1; ++s, ++o) {
        keys[o] = s;
        vals[o] = static_cast<uint32_t>(p);
    }
}

// slab-major SoA (the stable sort keeps each slab's entries in min-a order),
// each entry's slab and its box's first slab, per-slab segment ends
__global__ void k_slab_gather(const uint32_t* keys, const uint32_t* vals, unsigned long long E,
                              const SlabParams* Pp, const float* smin_a, const float* smax_a, const float4* sbox,
                              const uint4* svid, const uint2* sq, float* emin_a, float* emax_a, float4* ebox,
                              uint4* evid, uint2* equant, uint32_t* eslab, uint32_t* efirst, uint32_t* slab_end)
{
    const unsigned long long e = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (e >= E)
        return;
    const SlabParams P = *Pp;
    const uint32_t p = vals[e], s = keys[e];
    const float4 b = sbox[p];
    emin_a[e] = smin_a[p];
    emax_a[e] = smax_a[p];
    ebox[e] = b;
    evid[e] = svid[p];
    equant[e] = sq[p];
    eslab[e] = s;
    efirst[e] = slab_of(P, P.side ? b.z : b.x);
    if (e + 1 == E || keys[e + 1] != s)
        slab_end[s] = static_cast<uint32_t>(e + 1);
}

__global__ void k_entry_len(const uint32_t* run_end, unsigned long long E, unsigned long long* len)
{
    const unsigned long long e = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (e < E)
        len[e] = run_end[e] - e - 1;
}

// K4 per entry: the window ends at the first entry of the same slab whose
// min-a exceeds this entry's max-a
__global__ void __launch_bounds__(kSumBlock) k_slab_run_ends(const float* emin_a, const float* emax_a, const uint32_t* eslab,
                                const uint32_t* slab_end, unsigned long long E, uint32_t* run_end,
                                unsigned long long* pair_tests)
{
    const unsigned long long e = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    unsigned long long len = 0;
    if (e < E) {
        const float reach = emax_a[e];
        unsigned long long a = e + 1, b = slab_end[eslab[e]];
        while (a < b) {
            const unsigned long long m = (a + b) >> 1;
            if (emin_a[m] <= reach)
                a = m + 1;
            else
                b = m;
        }
        run_end[e] = static_cast<uint32_t>(a);
        len = a - e - 1;
    }
    block_add(pair_tests, len);
}

// ---- stats: StqStats::round_sizes[r] = #{i : run_len(i) >= r+1}

__global__ void k_run_hist(const unsigned long long* run_len, unsigned long long k,
                           unsigned long long* hist, unsigned long long* max_run)
{
    const unsigned long long p = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (p >= k)
        return;
    const unsigned long long l = run_len[p];
    if (l) {
        atomicAdd(&hist[l], 1ull);
        atomicMax(max_run, l);
    }
}

__global__ void k_reverse(const unsigned long long* in, unsigned long long n, unsigned long long off,
                          unsigned long long* out)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i < n)
        out[i] = in[off - i];
}

template <typename T>
T* grow(DevBuf& b, uint64_t n)
{
    return static_cast<T*>(b.ensure(n * sizeof(T)));
}

template <typename F>
void cub_call(Ctx& c, F&& f)
{
    size_t bytes = 0;
    CCDK_CUDA_CHECK(f(nullptr, bytes));
    void* tmp = c.cub_tmp.ensure(bytes);
    CCDK_CUDA_CHECK(f(tmp, bytes));
}

} // namespace

void broad_phase(Ctx& c, const BroadIn& in, BroadOut& out)
{
    cudaStream_t s = c.stream;
    const uint64_t k = in.k;
    out = BroadOut {};
    c.last_n_pairs = 0;
    c.last_rounds.clear();
    if (k < 2)
        return; // no pairs (broadphase.cpp:74-76; bf has no j > i either)
    if (k >= 0xffffffffull)
        throw Error(CCDK_CONFIG, "broad phase: more than 2^32-2 boxes");

    cudaEvent_t ev[4];
    for (int i = 0; i < 4; ++i)
        ev[i] = c.events.get(EventPool::kBroad + i);
    CCDK_CUDA_CHECK(cudaEventRecord(ev[0], s));

    auto* ctr = static_cast<DevCounters*>(c.counters.ensure(sizeof(DevCounters)));
    // clear the sweep counters; `error` belongs to the box build and is kept
    CCDK_CUDA_CHECK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), s));
    CCDK_CUDA_CHECK(cudaMemsetAsync(ctr->misc, 0, sizeof ctr->misc, s));

    // K2 choose_axis
    // d_axis[0] = axis, [1] = near tie (serial recomputation needed), [2] = serial ran
    int* d_axis = static_cast<int*>(c.axis.ensure(64));
    double* part = grow<double>(c.partials, 9 * kRedBlocks);
    CCDK_CUDA_CHECK(cudaMemsetAsync(d_axis, 0, 4 * sizeof(int), s));
    ++out.launches;
    k_axis_sum<<<kRedBlocks, kRedThreads, 0, s>>>(in.bmin, in.bmax, k, part);
    ++out.launches;
    k_axis_var<<<kRedBlocks, kRedThreads, 0, s>>>(in.bmin, in.bmax, k, part, part + 3 * kRedBlocks);
    ++out.launches;
    k_axis_pick<<<1, kRedThreads, 0, s>>>(part, k, d_axis);
    // The candidate set does not depend on the axis; the axis is observable
    // only through choose_axis itself, StqStats and SweepRange slices (and the
    // budget batching built on them), so the exact serial order is enforced
    // where those are requested.
    if (in.exact_axis) {
        ++out.launches;
        k_axis_serial<<<1, 96, 0, s>>>(in.bmin, in.bmax, k, d_axis);
    }
    CCDK_LAUNCH_CHECK();

    // K3 sort + permute
    uint32_t* keys_in = grow<uint32_t>(c.sort_keys_in, k);
    uint32_t* keys_out = grow<uint32_t>(c.sort_keys_out, k);
    uint32_t* vals_in = grow<uint32_t>(c.sort_vals_in, k);
    uint32_t* order = grow<uint32_t>(c.sort_vals_out, k);
    ++out.launches;
    k_sort_keys<<<grid_for(k, 256), 256, 0, s>>>(in.bmin, k, d_axis, keys_in, vals_in);
    CCDK_LAUNCH_CHECK();
    cub_call(c, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, keys_in, keys_out, vals_in, order,
                                               static_cast<int64_t>(k), 0, 32, s);
    });
    float* smin_a = grow<float>(c.smin_a, k);
    float* smax_a = grow<float>(c.smax_a, k);
    float4* sbox = grow<float4>(c.sbox, k);
    uint4* svid = grow<uint4>(c.svid, k);
    const bool bf = in.method == CCDK_BROAD_BF;
    uint32_t* sraw = bf ? grow<uint32_t>(c.raw, 2 * k) + k : nullptr;
    unsigned* qb = static_cast<unsigned*>(c.qbounds.ensure(8 * sizeof(unsigned)));
    CCDK_CUDA_CHECK(cudaMemsetAsync(qb, 0xff, 3 * sizeof(unsigned), s));
    CCDK_CUDA_CHECK(cudaMemsetAsync(qb + 3, 0, 3 * sizeof(unsigned), s));
    ++out.launches;
    k_quant_bounds<<<kRedBlocks, kRedThreads, 0, s>>>(in.bmin, in.bmax, k, qb);
    uint2* sq = grow<uint2>(c.squant, k);
    ++out.launches;
    k_permute<<<grid_for(k, 256), 256, 0, s>>>(in.bmin, in.bmax, in.vids, in.raw, k, d_axis, order,
                                               smin_a, smax_a, sbox, svid, sraw, qb, sq);
    CCDK_LAUNCH_CHECK();
    CCDK_CUDA_CHECK(cudaEventRecord(ev[1], s));

    // K4 run ends over the left range (stq/sap: sorted positions; bf: all,
    // filtered by raw position at emission)
    uint64_t lo = 0, hi = k - 1;
    if (!bf) {
        lo = std::min<uint64_t>(in.range_begin, k - 1);
        hi = std::min<uint64_t>(in.range_end, k - 1);
    }
    // rows of the sweep: the k sorted boxes, or in slab mode the E slab entries
    uint64_t rows = k;
    const float* w_min = smin_a;
    const float* w_max = smax_a;
    const float4* w_box = sbox;
    const uint4* w_vid = svid;
    const uint2* w_q = sq;
    const uint32_t* w_slab = nullptr;
    const uint32_t* w_first = nullptr;
    unsigned long long* d_range = &ctr->misc[0]; // misc[0..1]
    uint32_t* run_end = nullptr;
    // CCDK_SLAB=0 / =1 forces the 1-D / slab sweep; by default slab mode from
    // kSlabMinBoxes on (below it the set-up's ~10 launches and host read-back
    // cost more than the shorter windows save: C1, 75k boxes, 0.17 -> 0.24 ms)
    const char* slab_env = std::getenv("CCDK_SLAB"); // read per call: tests toggle it
    const bool slab_size_ok = slab_env ? slab_env[0] != '0' : k >= kSlabMinBoxes;
    const bool slab_try = !bf && in.allow_slab && slab_size_ok && lo == 0 && hi == k - 1 && !in.want_rounds
        && k < (uint64_t(1) << 30);
    if (slab_try) {
        char* par = static_cast<char*>(c.slab_par.ensure(64));
        double* sums = reinterpret_cast<double*>(par);
        SlabParams* P = reinterpret_cast<SlabParams*>(par + 16);
        CCDK_CUDA_CHECK(cudaMemsetAsync(sums, 0, 16, s));
        ++out.launches;
        k_slab_stats<<<kRedBlocks, kRedThreads, 0, s>>>(sbox, k, sums);
        const char* wf = std::getenv("CCDK_SLAB_W"); // slab width / mean box extent (tuning)
        ++out.launches;
        k_slab_params<<<1, 1, 0, s>>>(qb, d_axis, sums, k, wf ? std::atof(wf) : 2.0, P);
        uint32_t* cnt = grow<uint32_t>(c.slab_cnt, 2 * k);
        uint32_t* eoff = cnt + k;
        ++out.launches;
        k_slab_count<<<grid_for(k, 256), 256, 0, s>>>(sbox, k, P, cnt);
        CCDK_LAUNCH_CHECK();
        cub_call(c, [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, cnt, eoff, static_cast<int64_t>(k), s);
        });
        uint32_t tail[2];
        SlabParams hp {};
        unsigned long long berr = ~0ull;
        CCDK_CUDA_CHECK(cudaMemcpyAsync(&tail[0], eoff + k - 1, 4, cudaMemcpyDeviceToHost, s));
        CCDK_CUDA_CHECK(cudaMemcpyAsync(&tail[1], cnt + k - 1, 4, cudaMemcpyDeviceToHost, s));
        CCDK_CUDA_CHECK(cudaMemcpyAsync(&hp, P, sizeof hp, cudaMemcpyDeviceToHost, s));
        if (in.check_build_error)
            CCDK_CUDA_CHECK(cudaMemcpyAsync(&berr, &ctr->error, 8, cudaMemcpyDeviceToHost, s));
        CCDK_CUDA_CHECK(cudaStreamSynchronize(s));
        if (berr != ~0ull)
            throw Error(CCDK_INVALID_INPUT, "round_down_reduced: non-finite input");
        const uint64_t E = static_cast<uint64_t>(tail[0]) + tail[1];
        // copies of wide boxes multiply the entries; beyond 4 k the 1-D sweep wins
        if (hp.ok && E <= 4 * k) {
            uint32_t* ek = grow<uint32_t>(c.slab_keys, 2 * E);
            uint32_t* ev_ = grow<uint32_t>(c.slab_vals, 2 * E);
            ++out.launches;
            k_slab_emit<<<grid_for(k, 256), 256, 0, s>>>(sbox, k, P, eoff, ek, ev_);
            CCDK_LAUNCH_CHECK();
            cub_call(c, [&](void* t, size_t& b) { // stable: each slab stays in min-a order
                return cub::DeviceRadixSort::SortPairs(t, b, ek, ek + E, ev_, ev_ + E, static_cast<int64_t>(E),
                                                       0, 16, s);
            });
            float* emin = grow<float>(c.emin_a, E);
            float* emax = grow<float>(c.emax_a, E);
            float4* ebox = grow<float4>(c.ebox, E);
            uint4* evid = grow<uint4>(c.evid, E);
            uint2* eq = grow<uint2>(c.equant, E);
            uint32_t* eslab = grow<uint32_t>(c.eslab, 2 * E);
            uint32_t* efirst = eslab + E;
            uint32_t* slab_end = grow<uint32_t>(c.slab_end, hp.S);
            ++out.launches;
            k_slab_gather<<<grid_for(E, 256), 256, 0, s>>>(ek + E, ev_ + E, E, P, smin_a, smax_a, sbox, svid, sq,
                                                            emin, emax, ebox, evid, eq, eslab, efirst, slab_end);
            run_end = grow<uint32_t>(c.run_end, E);
            ++out.launches;
            k_slab_run_ends<<<grid_for(E, kSumBlock), kSumBlock, 0, s>>>(emin, emax, eslab, slab_end, E, run_end,
                                                              &ctr->pair_tests);
            if (in.shard_count > 1) {
                // multi-GPU: rank r sweeps the entry rows [B_r, B_{r+1}) that split
                // the total window length evenly (every pair has exactly one
                // emitting row, so any partition of rows partitions the pairs)
                unsigned long long* len = grow<unsigned long long>(c.prefix, 2 * E);
                ++out.launches;
                k_entry_len<<<grid_for(E, 256), 256, 0, s>>>(run_end, E, len);
                cub_call(c, [&](void* t, size_t& b) {
                    return cub::DeviceScan::InclusiveSum(t, b, len, len + E, static_cast<int64_t>(E), s);
                });
                ++out.launches;
                k_shard_range<<<1, 32, 0, s>>>(len + E, 0, E, in.shard_rank, in.shard_count, d_range);
            } else {
                ++out.launches;
                k_full_range<<<1, 1, 0, s>>>(0, E, d_range);
            }
            CCDK_LAUNCH_CHECK();
            rows = E;
            lo = 0;
            hi = E;
            w_min = emin;
            w_max = emax;
            w_box = ebox;
            w_vid = evid;
            w_q = eq;
            w_slab = eslab;
            w_first = efirst;
            out.slab_mode = true;
            out.slab_count = hp.S;
            out.slab_entries = E;
        }
    }
    const bool need_len = in.want_rounds || in.shard_count > 1;
    unsigned long long* run_len = nullptr;
    if (!out.slab_mode) {
        run_end = grow<uint32_t>(c.run_end, k);
        run_len = need_len ? grow<unsigned long long>(c.prefix, 2 * k) : nullptr;
        ++out.launches;
        k_run_ends<<<grid_for(k, kSumBlock), kSumBlock, 0, s>>>(smin_a, smax_a, k, lo, hi, run_end, run_len,
                                                     &ctr->pair_tests);
        CCDK_LAUNCH_CHECK();
        if (in.shard_count > 1) {
            unsigned long long* incl = run_len + k;
            cub_call(c, [&](void* t, size_t& b) {
                return cub::DeviceScan::InclusiveSum(t, b, run_len, incl, static_cast<int64_t>(k), s);
            });
            ++out.launches;
            k_shard_range<<<1, 32, 0, s>>>(incl, lo, hi, in.shard_rank, in.shard_count, d_range);
        } else {
            ++out.launches;
            k_full_range<<<1, 1, 0, s>>>(lo, hi, d_range);
        }
        CCDK_LAUNCH_CHECK();
    }
    // slab mode: long rows (boxes spanning a slab, e.g. a static floor) split
    // into short segments so no single warp walks thousands of hits
    const uint32_t cap = out.slab_mode ? kSlabCap : kCap, seg = out.slab_mode ? kSlabCap : kSeg;
    uint32_t* nseg = grow<uint32_t>(c.seg_off, 2 * rows);
    uint32_t* off = nseg + rows;
    ++out.launches;
    k_heavy_count<<<grid_for(rows, 256), 256, 0, s>>>(run_end, d_range, rows, nseg, cap, seg);
    cub_call(c, [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, nseg, off, static_cast<int64_t>(rows), s);
    });
    // segments total <= sum over rows of ceil(window / seg); grow on demand below
    uint64_t seg_cap = std::max<uint64_t>(c.segs.cap / sizeof(Seg), 1024);
    Seg* segs = grow<Seg>(c.segs, seg_cap);

    // StqStats round sizes
    if (in.want_rounds) {
        unsigned long long* hist = grow<unsigned long long>(c.rounds, 2 * (k + 1));
        CCDK_CUDA_CHECK(cudaMemsetAsync(hist, 0, (k + 1) * sizeof(unsigned long long), s));
        ++out.launches;
        k_run_hist<<<grid_for(k, 256), 256, 0, s>>>(run_len, k, hist, &ctr->misc[2]);
        CCDK_LAUNCH_CHECK();
    }

    // sizes needed on the host: heavy segment count (for the buffer) and max run
    unsigned long long host_ctr[8];
    auto read_ctr = [&]() {
        CCDK_CUDA_CHECK(cudaMemcpyAsync(host_ctr, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
        CCDK_CUDA_CHECK(cudaStreamSynchronize(s));
    };
    {
        // total heavy segments = off[k-1] + nseg[k-1]
        uint32_t tail[2];
        CCDK_CUDA_CHECK(cudaMemcpyAsync(&tail[0], off + rows - 1, 4, cudaMemcpyDeviceToHost, s));
        CCDK_CUDA_CHECK(cudaMemcpyAsync(&tail[1], nseg + rows - 1, 4, cudaMemcpyDeviceToHost, s));
        read_ctr();
        if (in.check_build_error && host_ctr[3] != ~0ull)
            throw Error(CCDK_INVALID_INPUT, "round_down_reduced: non-finite input");
        const uint64_t total = static_cast<uint64_t>(tail[0]) + tail[1];
        if (total > seg_cap) {
            seg_cap = total;
            segs = grow<Seg>(c.segs, seg_cap);
        }
    }
    out.pair_tests = host_ctr[1];
    if (in.want_rounds) {
        const uint64_t max_run = host_ctr[4 + 2];
        c.last_rounds.assign(max_run, 0);
        if (max_run) {
            unsigned long long* hist = c.rounds.as<unsigned long long>();
            unsigned long long* rev = hist + (k + 1);
            ++out.launches;
            k_reverse<<<grid_for(max_run, 256), 256, 0, s>>>(hist, max_run, max_run, rev);
            unsigned long long* scan = hist; // reuse: hist no longer needed after reversing
            cub_call(c, [&](void* t, size_t& b) {
                return cub::DeviceScan::InclusiveSum(t, b, rev, scan, static_cast<int64_t>(max_run), s);
            });
            // scan[i] = sum_{x >= max_run - i} hist[x] = round_sizes[max_run - 1 - i]
            ++out.launches;
            k_reverse<<<grid_for(max_run, 256), 256, 0, s>>>(scan, max_run, max_run - 1, rev);
            CCDK_LAUNCH_CHECK();
            CCDK_CUDA_CHECK(cudaMemcpyAsync(c.last_rounds.data(), rev, max_run * 8,
                                            cudaMemcpyDeviceToHost, s));
            CCDK_CUDA_CHECK(cudaStreamSynchronize(s));
        }
    }
    ++out.launches;
    k_heavy_gen<<<grid_for(rows, 256), 256, 0, s>>>(run_end, nseg, off, rows, segs, &ctr->n_heavy, cap, seg);
    CCDK_LAUNCH_CHECK();

    // K5 sweep (re-run once with a larger buffer if the candidate count overflows)
    const int nb = in.rank_bits ? in.rank_bits : ceil_log2(k);
    c.last_nb = nb;
    if (c.pair_capacity < 8 * k)
        c.pair_capacity = std::max<uint64_t>(8 * k, uint64_t(1) << 20);
    uint64_t n_pairs = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        unsigned long long* keys = grow<unsigned long long>(c.pair_keys, c.pair_capacity);
        CCDK_CUDA_CHECK(cudaMemsetAsync(&ctr->n_pairs, 0, 8, s));
        SweepArgs sa {};
        sa.smin_a = w_min;
        sa.smax_a = w_max;
        sa.sbox = w_box;
        sa.sq = w_q;
        sa.svid = w_vid;
        sa.slab = w_slab;
        sa.slab_first = w_first;
        sa.sraw = sraw;
        sa.run_end = run_end;
        sa.range = d_range;
        sa.row0 = lo;
        sa.k = rows;
        sa.nb = nb;
        sa.bf = bf;
        sa.bf_lo = in.range_begin;
        sa.bf_hi = in.range_end;
        sa.keys = keys;
        sa.cap = c.pair_capacity;
        sa.n_pairs = &ctr->n_pairs;
        sa.segs = segs;
        sa.n_heavy = &ctr->n_heavy;
        sa.short_len = out.slab_mode ? kShortLen : 0;
        sa.row_cap = cap;
        if (hi > lo) {
            const uint64_t warps = (hi - lo + kRowsPerWarp - 1) / kRowsPerWarp;
            ++out.launches;
            k_sweep_rows<<<grid_for(warps * 32, kRowsTB), kRowsTB, 0, s>>>(sa);
            if (sa.short_len) {
                ++out.launches;
                k_sweep_short<<<grid_for(hi - lo, kRowsTB), kRowsTB, 0, s>>>(sa);
            }
        }
        ++out.launches;
        k_sweep_heavy<<<4 * c.num_sms, kRowsTB, 0, s>>>(sa);
        CCDK_LAUNCH_CHECK();
        read_ctr();
        n_pairs = host_ctr[0];
        out.range_lo = host_ctr[4]; // the swept left range (shard slice)
        out.range_hi = host_ctr[5];
        if (n_pairs <= c.pair_capacity)
            break;
        c.pair_capacity = n_pairs + n_pairs / 4;
    }
    CCDK_CUDA_CHECK(cudaEventRecord(ev[2], s));

    // K6 canonical order
    unsigned long long* sorted = grow<unsigned long long>(c.pair_keys_sorted, std::max<uint64_t>(n_pairs, 1));
    if (n_pairs) {
        unsigned long long* keys = c.pair_keys.as<unsigned long long>();
        cub_call(c, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, keys, sorted, static_cast<int64_t>(n_pairs),
                                                  0, 2 * nb, s);
        });
        if (in.unique) {
            unsigned long long* nsel = &ctr->misc[3];
            cub_call(c, [&](void* t, size_t& b) {
                return cub::DeviceSelect::Unique(t, b, sorted, keys, nsel, static_cast<int64_t>(n_pairs), s);
            });
            read_ctr();
            n_pairs = host_ctr[4 + 3];
            CCDK_CUDA_CHECK(cudaMemcpyAsync(sorted, keys, n_pairs * 8, cudaMemcpyDeviceToDevice, s));
        }
    }
    CCDK_CUDA_CHECK(cudaEventRecord(ev[3], s));
    int* axis_h = static_cast<int*>(c.pin_axis.ensure(64)); // words 0-3 axis, 8-byte word 4: the step's VF count
    CCDK_CUDA_CHECK(cudaMemcpyAsync(axis_h, d_axis, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
    out.n_pairs = n_pairs;
    c.last_n_pairs = n_pairs;
    if (!in.defer_collect)
        broad_collect(c, out);
}

// Stage times and the axis of the last broad phase (waits for its end).
void broad_collect(Ctx& c, BroadOut& out)
{
    cudaEvent_t ev[4];
    for (int i = 0; i < 4; ++i)
        ev[i] = c.events.get(EventPool::kBroad + i);
    CCDK_CUDA_CHECK(cudaEventSynchronize(ev[3]));
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&out.ms_axis_sort, ev[0], ev[1]));
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&out.ms_sweep, ev[1], ev[2]));
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&out.ms_pairsort, ev[2], ev[3]));
    const int* axis = c.pin_axis.as<int>();
    out.axis = axis[0];
    out.axis_near_tie = axis[1] != 0;
    out.axis_serial = axis[2] != 0;
}

} // namespace ccdk
