// K7 classify, K8 breadth-first interval narrow phase, K9 reduction.
//
// Reference: proj/src/narrowphase.cpp:189-311 (narrow_phase) and
// proj/src/broadphase.cpp:194-239 (classify).
//
// K8 keeps the reference's schedule semantics exactly (SURVEY §7 "hard
// parts"): whole generations; pruning against a per-query ToI SNAPSHOT taken
// at the generation start (a dirty list refreshes only queries whose ToI
// dropped); per-query split budget counted per generation (an atomic request
// counter: the first max_splits requests are admitted, any later one folds
// its t.lo and marks the query exhausted, and the exhausted query's admitted
// children are folded and dropped at the start of the next generation).  All
// of these are order-independent, so unordered atomic appends reproduce the
// reference's serial fold bit for bit.
//
// Interval records are compact SoA: query id, (t,u,v).lo as doubles and the
// three bisection depths packed in a u64; hi = lo + 2^-depth exactly.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ccdk_internal.cuh"
#include "ccdk_interval.cuh"

namespace ccdk {

namespace {

constexpr unsigned kNoGen = 0xffffffffu;
constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
constexpr int kGenBlock = 128;
constexpr unsigned kMaxGens = 4096; // > the 4000-generation guard
#ifndef CCDK_GEN_UNROLL
#define CCDK_GEN_UNROLL 8
#endif
constexpr int kGenUnroll = CCDK_GEN_UNROLL; // generations per WHILE iteration of the graph
#ifndef CCDK_PDL
#define CCDK_PDL 1
#endif
constexpr bool kUsePdl = CCDK_PDL != 0; // programmatic dependent launch inside the generation chain
#ifndef CCDK_DEFER_APPEND
#define CCDK_DEFER_APPEND 0
#endif
#ifndef CCDK_GEN_MINB
#define CCDK_GEN_MINB 3
#endif

// Interval storage.  Every split appends ONE record — the split interval
// itself (query id, (t,u,v).lo, packed depths) — to the region of its split
// dimension; the record stands for its two children (lower and upper half
// along that dimension, narrowphase.cpp:122-132), which the next generation
// evaluates together (iv::process_pair).  Generation 0 evaluates the roots
// [0,1]^3 (one per query, implicit).
struct Region {
    uint32_t* qid;
    double* t;
    double* u;
    double* v;
    unsigned long long* dep;
};

struct GenArgs {
    uint32_t* qf;      // per-query kind | exact-widening flag (iv::kKind*)
    const uint8_t* kind;
    const double* pts;
    const double* sep;
    double sep_default;
    iv::Cfg cfg;
    unsigned long long max_splits;
    unsigned long long* toi;
    unsigned long long* snap;
    unsigned long long* splits;
    unsigned* exh_gen;
    uint8_t* zdiag;
    unsigned* dirty;                 // queries whose ToI dropped (duplicates allowed)
    Region reg[2][3];                // [generation parity][split dimension]
    unsigned long long cap_pairs;    // records per region buffer
    unsigned long long sem_cap;      // queue_capacity (narrowphase.cpp:299-302); ~0 = unbounded
    unsigned long long gen_stop;     // stop after this generation (~0 = run to the end)
    NarrowScalars* sc;
    cudaGraphConditionalHandle cond; // WHILE node of the generation graph
    unsigned long long* gen_sizes;   // compacted queue size per generation (kMaxGens entries)
};

__device__ __forceinline__ unsigned long long dbits(double x)
{
    return static_cast<unsigned long long>(__double_as_longlong(x));
}

__device__ __forceinline__ void warp_add(unsigned long long* dst, unsigned v)
{
    const unsigned s = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && s)
        atomicAdd(dst, static_cast<unsigned long long>(s));
}

// L2 eviction priority of the generation's loads (CCDK_REC_POLICY, A/B
// switch): 1 = query records evict_last (re-read by the query's next
// intervals one generation later), 2 = plus the interval records of the
// current generation evict_first (dead after this read).
#ifndef CCDK_REC_POLICY
#define CCDK_REC_POLICY 2
#endif
__device__ __forceinline__ unsigned long long policy_evict_last()
{
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_first()
{
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8_hint(void* smem, const void* gmem, unsigned long long pol)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
                 : "memory");
}
// 16-byte copies through L1 (.ca) or L2 only (.cg)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool l1)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if (l1)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, bool l1, unsigned long long pol)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if (l1)
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
                     : "memory");
    else
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
                     : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Collision of one interval: fold its t.lo into the query's live ToI and
// queue the query for the snapshot refresh (cand = t.lo < the snapshot, else
// the box would have been pruned, so the ToI drops this generation).
__device__ __forceinline__ void record_collision(const GenArgs& a, unsigned q, double cand, bool zd)
{
    atomicMin(&a.toi[q], dbits(cand));
    const unsigned long long slot = atomicAdd(&a.sc->dirty_n, 1ull);
    if (slot < a.sc->dirty_cap)
        a.dirty[slot] = q;
    if (zd)
        a.zdiag[q] = 1;
}

// Split records of this batch: per lane up to two (one per child), each
// appended to the region of its split dimension with one warp-aggregated
// cursor atomic per region.
struct SplitRec {
    int dim; // -1: none
    double tlo, ulo, vlo;
    unsigned long long dp;
};

// The three cursor atomics are one instruction (lane d bumps region d), so
// the warp waits for one atomic round trip per batch, not up to three.
__device__ __forceinline__ void append_splits(const GenArgs& a, int nb, unsigned lane, unsigned q,
                                              const SplitRec r[2])
{
    const unsigned lt = (1u << lane) - 1;
    unsigned off[2] = {0, 0}; // slot of each child within its region's share
    unsigned my_cnt = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const unsigned m0 = __ballot_sync(0xffffffffu, r[0].dim == d);
        const unsigned m1 = __ballot_sync(0xffffffffu, r[1].dim == d);
        if (r[0].dim == d)
            off[0] = __popc(m0 & lt);
        if (r[1].dim == d)
            off[1] = __popc(m0) + __popc(m1 & lt);
        if (lane == static_cast<unsigned>(d))
            my_cnt = __popc(m0) + __popc(m1);
    }
    if (!__any_sync(0xffffffffu, my_cnt != 0))
        return;
    unsigned long long base = 0;
    if (my_cnt)
        base = atomicAdd(&a.sc->next_pairs[lane], static_cast<unsigned long long>(my_cnt));
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
        const int d = r[ch].dim;
        const unsigned long long b = __shfl_sync(0xffffffffu, base, d < 0 ? 0 : d);
        if (d < 0)
            continue;
        const unsigned long long slot = b + off[ch];
        const Region& R = a.reg[nb][d];
        if (slot < a.cap_pairs) {
            R.qid[slot] = q;
            R.t[slot] = r[ch].tlo;
            R.u[slot] = r[ch].ulo;
            R.v[slot] = r[ch].vlo;
            R.dep[slot] = r[ch].dp;
        } else {
            a.sc->phys_overflow = 1;
        }
    }
}

#if CCDK_DEFER_APPEND
// The same append in two halves (CCDK_DEFER_APPEND): the cursor atomic is
// issued at the end of a batch and its result consumed only after the next
// batch's loads are issued, so the atomic's round trip overlaps the loop
// head instead of stalling the shuffle right behind it.
__device__ __forceinline__ void append_reserve(const GenArgs& a, unsigned lane, const SplitRec r[2], unsigned off[2],
                                               unsigned long long& base)
{
    const unsigned lt = (1u << lane) - 1;
    off[0] = off[1] = 0;
    unsigned my_cnt = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const unsigned m0 = __ballot_sync(0xffffffffu, r[0].dim == d);
        const unsigned m1 = __ballot_sync(0xffffffffu, r[1].dim == d);
        if (r[0].dim == d)
            off[0] = __popc(m0 & lt);
        if (r[1].dim == d)
            off[1] = __popc(m0) + __popc(m1 & lt);
        if (lane == static_cast<unsigned>(d))
            my_cnt = __popc(m0) + __popc(m1);
    }
    base = 0;
    if (my_cnt)
        base = atomicAdd(&a.sc->next_pairs[lane], static_cast<unsigned long long>(my_cnt));
}

__device__ __forceinline__ void append_write(const GenArgs& a, int nb, unsigned q, const SplitRec r[2],
                                             const unsigned off[2], unsigned long long base)
{
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
        const int d = r[ch].dim;
        const unsigned long long b = __shfl_sync(0xffffffffu, base, d < 0 ? 0 : d);
        if (d < 0)
            continue;
        const unsigned long long slot = b + off[ch];
        const Region& R = a.reg[nb][d];
        if (slot < a.cap_pairs) {
            R.qid[slot] = q;
            R.t[slot] = r[ch].tlo;
            R.u[slot] = r[ch].ulo;
            R.v[slot] = r[ch].vlo;
            R.dep[slot] = r[ch].dp;
        } else {
            a.sc->phys_overflow = 1;
        }
    }
}
#endif

// ---- generation 0: the roots [0,1]^3, one thread per query, coordinates
// read straight from the query record (one generation of the ~80).
__global__ void __launch_bounds__(kGenBlock) k_gen0(GenArgs a)
{
    NarrowScalars* sc = a.sc;
    const unsigned lane = threadIdx.x & 31;
    unsigned evals = 0, split_actions = 0;
    const unsigned long long n = sc->nq;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    // warp-uniform trip count (the append is warp-collective)
    const unsigned long long n_up = (n + 31) & ~31ull;
    for (unsigned long long q0 = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         q0 < n_up; q0 += stride) {
        const bool valid = q0 < n;
        const unsigned q = static_cast<unsigned>(valid ? q0 : 0);
        SplitRec r[2];
        r[0].dim = r[1].dim = -1;
        if (valid) {
            const iv::Box bx { 0.0, 1.0, 0.0, 1.0, 0.0, 1.0 };
            const unsigned qf = a.qf[q];
            const bool vf = !(qf & iv::kKindEE);
            const double sep = a.sep ? a.sep[q] : a.sep_default;
            const iv::GlobalPtsIL P { a.pts + 24ull * q };
            double cand = 0;
            bool zd = false, evald = false;
            int dim = -1, act;
            if (!(qf & iv::kKindExact)) {
                act = iv::process_one<iv::Fast>(vf, P, bx, CUDART_INF, sep, a.cfg, cand, zd, dim, evald);
            } else {
                const iv::Outcome o = iv::process_exact<iv::GlobalPtsIL>(vf, P, bx, CUDART_INF, sep, a.cfg);
                act = o.act;
                cand = o.cand;
                zd = o.zdiag;
                dim = o.dim;
                evald = o.evaluated;
            }
            evals += evald;
            if (act == iv::kCollision) {
                record_collision(a, q, cand, zd);
            } else if (act == iv::kSplit) {
                ++split_actions;
                // t.lo == 0 here: exempt from the budget in no-zero-ToI mode.
                // A root is its query's only request of generation 0 and
                // max_splits >= 1, so it is always admitted (no read-back).
                if (!a.cfg.no_zero_toi)
                    atomicAdd(&a.splits[q], 1ull);
                r[0] = { dim, 0.0, 0.0, 0.0, 0ull };
            }
        }
        append_splits(a, 1, lane, q, r);
    }
    warp_add(&sc->evaluations, evals);
    warp_add(&sc->split_actions, split_actions);
}

// ---- generations >= 1: one lane per split record (= a sibling pair).
//
// Per-warp shared-memory stage, element-major (element e of lane l at
// [32 e + l]): the query coordinates (24 doubles), the record (t, u, v lo,
// depths), and the per-query scalars (snapshot ToI, separation, exhausted
// generation | query flags), all brought in by cp.async while the previous
// batch is evaluated; the next batch's query ids ride one batch ahead.
constexpr int kStageDoubles = 24 * 32;
constexpr int kMetaDoubles = 7 * 32;
constexpr int kQidDoubles = 16;
constexpr int kWarpSmemDoubles = 2 * kStageDoubles + kMetaDoubles + kQidDoubles;
constexpr int kGenSmem = (kGenBlock / 32) * kWarpSmemDoubles * sizeof(double);
enum { kMT = 0, kMU, kMV, kMDep, kMSnap, kMExh, kMSplits };

struct BatchLoc {
    int d;                    // region (split dimension)
    unsigned long long i0;    // first record of the batch
    unsigned long long n;     // records in the region
};

// Batch b of the concatenated region batch space (regions padded to whole
// batches so a batch's split dimension is warp-uniform).  Scalar selects, no
// runtime-indexed arrays (those would live in local memory).
__device__ __forceinline__ BatchLoc locate(unsigned long long nb0, unsigned long long nb1,
                                           unsigned long long c0, unsigned long long c1,
                                           unsigned long long c2, unsigned long long b)
{
    BatchLoc L;
    if (b < nb0) {
        L.d = 0;
        L.n = c0;
    } else if (b < nb0 + nb1) {
        L.d = 1;
        L.n = c1;
        b -= nb0;
    } else {
        L.d = 2;
        L.n = c2;
        b -= nb0 + nb1;
    }
    L.i0 = b << 5;
    return L;
}

__device__ __forceinline__ const Region& region(const GenArgs& a, int par, int d)
{
    return d == 0 ? a.reg[par][0] : d == 1 ? a.reg[par][1] : a.reg[par][2];
}

template <int D>
__device__ __forceinline__ iv::PairOutcome eval_pair(bool vf, const iv::SmemPts& P, const iv::PairBox& pb,
                                                     const bool alive[2], double sep, const iv::Cfg& cfg)
{
    return iv::process_pair<D, iv::SmemPts>(vf, P, pb, alive, sep, cfg);
}

__global__ void __launch_bounds__(kGenBlock, CCDK_GEN_MINB) k_generation(GenArgs a)
{
    cudaGridDependencySynchronize(); // PDL: the previous finish has completed (no-op otherwise)
    extern __shared__ double gsm[];
    NarrowScalars* sc = a.sc;
    if (!sc->cont)
        return;
    const unsigned gen = static_cast<unsigned>(sc->gen);
    const int cb = gen & 1, nb = cb ^ 1;
    const unsigned long long c0 = sc->cur_pairs[0], c1 = sc->cur_pairs[1], c2 = sc->cur_pairs[2];
    const unsigned long long nb0 = (c0 + 31) >> 5, nb1 = (c1 + 31) >> 5, nb2 = (c2 + 31) >> 5;
    const unsigned long long nbatch = nb0 + nb1 + nb2;

    const unsigned lane = threadIdx.x & 31;
    const unsigned wib = threadIdx.x >> 5;
    double* stage0 = gsm + wib * kWarpSmemDoubles;
    double* meta = stage0 + 2 * kStageDoubles;
    unsigned* qbuf = reinterpret_cast<unsigned*>(meta + kMetaDoubles);
    const unsigned long long W = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long b = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x >> 5) + wib;
    unsigned evals = 0, split_actions = 0, dropped = 0;
#ifdef CCDK_STATS
    unsigned st_pairs = 0, st_single = 0;
#endif
    if (b >= nbatch)
        return; // warp-uniform; no __syncthreads in this kernel

#if CCDK_REC_POLICY >= 1
    const unsigned long long pol_keep = policy_evict_last();
#endif
#if CCDK_REC_POLICY >= 2
    const unsigned long long pol_dead = policy_evict_first();
#endif
    auto issue = [&](unsigned long long bb, unsigned q, int st) {
        // batch bb's coordinates + record + query scalars, batch bb+W's ids
        if (bb < nbatch) {
            const BatchLoc L = locate(nb0, nb1, c0, c1, c2, bb);
            const unsigned long long i = L.i0 + lane;
            // Query records through L1 (.ca) when any two neighbouring lanes
            // of the batch share a query (dense BFS trees: C3/C5, measured
            // 5-25% faster through L1), otherwise L2-only copies (.cg; C2/C4,
            // where L1 allocation only costs: 8% faster).
            const unsigned q_prev = __shfl_up_sync(0xffffffffu, q, 1); // all lanes: no divergence
            const bool dup = lane > 0 && i < L.n && q_prev == q;
#ifndef CCDK_L1_DUP
#define CCDK_L1_DUP 1
#endif
#ifdef CCDK_L1
            const bool l1_records = CCDK_L1;
#else
            const bool l1_records = __popc(__ballot_sync(0xffffffffu, dup)) >= CCDK_L1_DUP;
#endif
            if (i < L.n) {
                const Region& R = region(a, cb, L.d);
                // the record's 12 (x0, x1) pairs (internal order), pair-major
                double* coords = stage0 + st * kStageDoubles;
                const double* src = a.pts + 24ull * q;
#if CCDK_REC_POLICY >= 1
#pragma unroll
                for (int k = 0; k < 12; ++k)
                    cp_async16_hint(coords + 64 * k + 2 * lane, src + 2 * k, l1_records, pol_keep);
#else
#pragma unroll
                for (int k = 0; k < 12; ++k)
                    cp_async16(coords + 64 * k + 2 * lane, src + 2 * k, l1_records);
#endif
#if CCDK_REC_POLICY >= 2
                cp_async8_hint(meta + 32 * kMT + lane, R.t + i, pol_dead);
                cp_async8_hint(meta + 32 * kMU + lane, R.u + i, pol_dead);
                cp_async8_hint(meta + 32 * kMV + lane, R.v + i, pol_dead);
                cp_async8_hint(meta + 32 * kMDep + lane, R.dep + i, pol_dead);
#else
                cp_async8(meta + 32 * kMT + lane, R.t + i);
                cp_async8(meta + 32 * kMU + lane, R.u + i);
                cp_async8(meta + 32 * kMV + lane, R.v + i);
                cp_async8(meta + 32 * kMDep + lane, R.dep + i);
#endif
                cp_async8(meta + 32 * kMSnap + lane, a.snap + q);
                unsigned* ex = reinterpret_cast<unsigned*>(meta + 32 * kMExh + lane);
                cp_async4(ex, a.exh_gen + q);
                cp_async4(ex + 1, a.qf + q);
                cp_async8(meta + 32 * kMSplits + lane, a.splits + q);
            }
        }
        if (bb + W < nbatch) {
            const BatchLoc L = locate(nb0, nb1, c0, c1, c2, bb + W);
            const unsigned long long i = L.i0 + lane;
            if (i < L.n)
                cp_async4(qbuf + lane, region(a, cb, L.d).qid + i);
        }
        cp_async_commit();
    };

    // every query makes at most 2 split requests per record of this
    // generation, so at most req_bound in total this generation
    const unsigned long long req_bound = 2 * (c0 + c1 + c2);
    unsigned q_cur;
    {
        const BatchLoc L = locate(nb0, nb1, c0, c1, c2, b);
        const unsigned long long i = L.i0 + lane;
        q_cur = i < L.n ? region(a, cb, L.d).qid[i] : 0u;
    }
    issue(b, q_cur, 0);
    int st = 0;
#if CCDK_DEFER_APPEND
    SplitRec pr[2]; // split records of the previous batch, appended after the next issue
    pr[0].dim = pr[1].dim = -1;
    unsigned poff[2] = { 0, 0 };
    unsigned long long pbase = 0;
    unsigned pq = 0;
#endif

    for (; b < nbatch; b += W) {
        cp_async_wait<0>(); // batch b's data and batch b+W's ids (issued one batch ago)
        const BatchLoc L = locate(nb0, nb1, c0, c1, c2, b);
        const bool valid = L.i0 + lane < L.n;
        const unsigned q = q_cur;
        const double tlo = meta[32 * kMT + lane];
        const double ulo = meta[32 * kMU + lane];
        const double vlo = meta[32 * kMV + lane];
        const unsigned long long dp = static_cast<unsigned long long>(__double_as_longlong(meta[32 * kMDep + lane]));
        const double t_star = meta[32 * kMSnap + lane];
        const unsigned exh = reinterpret_cast<const unsigned*>(meta + 32 * kMExh + lane)[0];
        const unsigned qf = reinterpret_cast<const unsigned*>(meta + 32 * kMExh + lane)[1];
        const unsigned long long splits0 =
            static_cast<unsigned long long>(__double_as_longlong(meta[32 * kMSplits + lane]));
        q_cur = qbuf[lane];
        // batch b+W streams into the other coordinate buffer while b is evaluated
        issue(b + W, q_cur, st ^ 1);
#if CCDK_DEFER_APPEND
        append_write(a, nb, pq, pr, poff, pbase); // the previous batch's split records
#endif

        SplitRec r[2];
        r[0].dim = r[1].dim = -1;
        unsigned req = 0;
        if (valid) {
            const int D = L.d;
            if (exh < gen) {
                // exhausted in an earlier generation: fold the children's
                // min t.lo (= the record's t.lo) and drop both
                // (narrowphase.cpp:280-291)
                atomicMin(&a.toi[q], dbits(tlo));
                if (a.cfg.no_zero_toi && tlo == 0.0)
                    a.zdiag[q] = 1;
                dropped += 2;
            } else {
                // the pair's samples: (lo, mid, hi) along D, (lo, hi) elsewhere
                const unsigned dD = (dp >> (16 * D)) & 0xffff;
                iv::PairBox pb;
                const double wt = iv::dyadic_width(dp & 0xffff);
                const double wu = iv::dyadic_width((dp >> 16) & 0xffff);
                const double wv = iv::dyadic_width((dp >> 32) & 0xffff);
                pb.t[0] = tlo;
                pb.u[0] = ulo;
                pb.v[0] = vlo;
                // split_box (narrowphase.cpp:122-132): the exact dyadic midpoint
                const double mid = __dadd_rn(D == 0 ? tlo : D == 1 ? ulo : vlo, iv::dyadic_width(dD + 1));
                pb.t[1] = D == 0 ? mid : __dadd_rn(tlo, wt);
                pb.t[2] = __dadd_rn(tlo, wt);
                pb.u[1] = D == 1 ? mid : __dadd_rn(ulo, wu);
                pb.u[2] = __dadd_rn(ulo, wu);
                pb.v[1] = D == 2 ? mid : __dadd_rn(vlo, wv);
                pb.v[2] = __dadd_rn(vlo, wv);
                const bool vf = !(qf & iv::kKindEE);
                bool alive[2];
                double clo[2][3];
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    clo[ch][0] = (D == 0 && ch) ? mid : tlo;
                    clo[ch][1] = (D == 1 && ch) ? mid : ulo;
                    clo[ch][2] = (D == 2 && ch) ? mid : vlo;
                    // process_interval's pre-evaluation prunes (narrowphase.cpp:138-143)
                    alive[ch] = !(clo[ch][0] >= t_star || clo[ch][0] >= a.cfg.t_max)
                        && !(vf && __dadd_rn(clo[ch][1], clo[ch][2]) > 1.0);
                }
#ifdef CCDK_STATS
                st_pairs += (alive[0] || alive[1]);
                st_single += (alive[0] != alive[1]);
#endif
                if (alive[0] || alive[1]) {
                    // per-query separation (Relative min-separation mode only)
                    const double sep = a.sep ? a.sep[q] : a.sep_default;
                    const iv::SmemPts P { stage0 + st * kStageDoubles + 2 * lane };
                    iv::PairOutcome o;
                    if (!(qf & iv::kKindExact)) {
                        if (D == 0)
                            o = eval_pair<0>(vf, P, pb, alive, sep, a.cfg);
                        else if (D == 1)
                            o = eval_pair<1>(vf, P, pb, alive, sep, a.cfg);
                        else
                            o = eval_pair<2>(vf, P, pb, alive, sep, a.cfg);
                    } else {
#pragma unroll
                        for (int ch = 0; ch < 2; ++ch) {
                            o.act[ch] = iv::kPruned;
                            o.evaluated[ch] = false;
                            if (!alive[ch])
                                continue;
                            // child box: lower half [lo, mid] or upper half [mid, hi] along D
                            const iv::Box bx { clo[ch][0], (D == 0 && !ch) ? mid : __dadd_rn(tlo, wt),
                                               clo[ch][1], (D == 1 && !ch) ? mid : __dadd_rn(ulo, wu),
                                               clo[ch][2], (D == 2 && !ch) ? mid : __dadd_rn(vlo, wv) };
                            const iv::Outcome e = iv::process_exact<iv::SmemPts>(vf, P, bx, t_star, sep, a.cfg);
                            o.act[ch] = e.act;
                            o.cand[ch] = e.cand;
                            o.zdiag[ch] = e.zdiag;
                            o.dim[ch] = e.dim;
                            o.evaluated[ch] = e.evaluated;
                        }
                    }
                    const unsigned long long dpc = dp + (1ull << (16 * D));
                    unsigned counted = 0; // budget-counted split requests of the pair
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch) {
                        evals += o.evaluated[ch];
                        if (o.act[ch] == iv::kCollision) {
                            record_collision(a, q, o.cand[ch], o.zdiag[ch]);
                        } else if (o.act[ch] == iv::kSplit) {
                            ++split_actions;
                            counted += !(a.cfg.no_zero_toi && clo[ch][0] == 0.0);
                            r[ch] = { o.dim[ch], clo[ch][0], clo[ch][1], clo[ch][2], dpc };
                        }
                    }
                    req = counted;
                }
            }
        }
        // split budget (narrowphase.cpp:254-271): this pair's requests get
        // indices old .. old+req-1 and any index >= max_splits exhausts the
        // query.  splits0 (read after the generation started) + req_bound
        // bounds every index of this generation, so below the budget no
        // index can reach it and the count is a fire-and-forget reduction;
        // otherwise the exact old value decides.
        if (req) {
            if (splits0 + req_bound <= a.max_splits) {
                atomicAdd(&a.splits[q], static_cast<unsigned long long>(req));
            } else {
                const unsigned long long old = atomicAdd(&a.splits[q], static_cast<unsigned long long>(req));
                if (old + req > a.max_splits)
                    a.exh_gen[q] = gen;
            }
        }
#if CCDK_DEFER_APPEND
        append_reserve(a, lane, r, poff, pbase);
        pr[0] = r[0];
        pr[1] = r[1];
        pq = q;
#else
        append_splits(a, nb, lane, q, r);
#endif
        st ^= 1;
    }
#if CCDK_DEFER_APPEND
    append_write(a, nb, pq, pr, poff, pbase);
#endif
    cp_async_wait<0>();
    warp_add(&sc->evaluations, evals);
    warp_add(&sc->split_actions, split_actions);
    warp_add(&sc->dropped, dropped);
#ifdef CCDK_STATS
    warp_add(&sc->vf_count, st_pairs);       // diagnostics only: pairs with a live child
    warp_add(&sc->next_n, st_single);        // diagnostics only: pairs with exactly one live child
#endif
}

// Generation end: refresh snapshots of queries whose ToI dropped, then (last
// block) the queue bookkeeping of narrowphase.cpp:278-304.
//
// The reference tests next.size() > queue_capacity AFTER removing the
// children of queries exhausted in this generation (narrowphase.cpp:280-302),
// and on overflow returns the per-query results folded so far.  The split
// records of the next generation count raw children; when that raw count
// exceeds the capacity (or the run stops at gen_stop), every block scans the
// next generation's records once: children of exhausted queries are counted
// (the exact next.size()) and their t.lo folded into the query's ToI — the
// same fold the next generation would do when it drops them (idempotent).
__global__ void k_finish(GenArgs a)
{
    cudaGridDependencySynchronize(); // PDL: the generation kernel has completed (no-op otherwise)
    NarrowScalars* sc = a.sc;
    if (!sc->cont) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && a.cond)
            cudaGraphSetConditional(a.cond, 0u);
        return;
    }
    const unsigned long long nd = sc->dirty_n;
    const bool all = nd > sc->dirty_cap; // list overflowed: refresh every query
    const unsigned long long m = all ? sc->nq : nd;
    const unsigned long long tid = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    const unsigned long long nthreads = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long i = tid; i < m; i += nthreads) {
        const unsigned q = all ? static_cast<unsigned>(i) : a.dirty[i];
        a.snap[q] = a.toi[q];
    }
    const unsigned long long gen = sc->gen;
    const unsigned long long raw_pairs = sc->next_pairs[0] + sc->next_pairs[1] + sc->next_pairs[2];
    const bool scan = 2 * raw_pairs > a.sem_cap || gen == a.gen_stop;
    if (scan) {
        const int nb = static_cast<int>(gen & 1) ^ 1;
        unsigned cnt = 0;
        for (int d = 0; d < 3; ++d) {
            const Region& R = a.reg[nb][d];
            const unsigned long long nr = sc->next_pairs[d] < a.cap_pairs ? sc->next_pairs[d] : a.cap_pairs;
            for (unsigned long long i = tid; i < nr; i += nthreads) {
                const unsigned q = R.qid[i];
                if (a.exh_gen[q] != kNoGen) {
                    const double tlo = R.t[i];
                    atomicMin(&a.toi[q], dbits(tlo));
                    if (a.cfg.no_zero_toi && tlo == 0.0)
                        a.zdiag[q] = 1;
                    cnt += 2;
                }
            }
        }
        warp_add(&sc->exh_next, cnt);
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&sc->finish_ticket, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0)
        return;
    __threadfence();
    const unsigned long long compacted = sc->cur_n - sc->dropped;
    if (compacted > sc->peak)
        sc->peak = compacted;
    if (sc->gen < kMaxGens)
        a.gen_sizes[sc->gen] = compacted;
    unsigned long long raw_next = 0;
    for (int d = 0; d < 3; ++d) {
        const unsigned long long r = sc->next_pairs[d];
        raw_next += r;
        if (r > a.cap_pairs)
            sc->phys_overflow = 1;
        sc->cur_pairs[d] = r > a.cap_pairs ? a.cap_pairs : r;
        sc->next_pairs[d] = 0;
    }
    if (scan) {
        if (2 * raw_next - sc->exh_next > a.sem_cap) // narrowphase.cpp:299-302
            sc->sem_overflow = 1;
        if (gen == a.gen_stop)
            sc->stopped = 1;
        sc->exh_next = 0;
    }
    sc->gen += 1;
    sc->cur_n = 2 * (sc->cur_pairs[0] + sc->cur_pairs[1] + sc->cur_pairs[2]);
    sc->dirty_n = 0;
    sc->dropped = 0;
    sc->finish_ticket = 0;
    sc->cont = (raw_next > 0 && !sc->sem_overflow && !sc->phys_overflow && !sc->stopped) ? 1 : 0;
    // a BFS tree is at most 3 x 1075 bisections deep; more generations than
    // that means corrupted state, never a legitimate run
    if (sc->cont && sc->gen > 4000) {
        sc->cont = 0;
        sc->gen_limit = 1;
    }
    __threadfence();
    if (a.cond)
        cudaGraphSetConditional(a.cond, sc->cont ? 1u : 0u);
}

__global__ void k_init_scalars(NarrowScalars* sc, unsigned long long n)
{
    unsigned long long* w = reinterpret_cast<unsigned long long*>(sc);
    for (unsigned i = threadIdx.x; i < sizeof(NarrowScalars) / 8; i += blockDim.x)
        w[i] = 0;
    __syncwarp();
    if (threadIdx.x == 0) {
        sc->cur_n = n;
        sc->nq = n;
        sc->dirty_cap = 2 * n;
        sc->cont = 1;
        sc->global_toi_bits = kInfBits;
    }
}

__device__ __forceinline__ uint32_t query_flags(uint8_t kind, const double* pts)
{
    return static_cast<uint32_t>((kind == CCDK_QUERY_EE ? iv::kKindEE : 0)
                                 | (iv::fast_ok(iv::GlobalPts { pts }) ? 0 : iv::kKindExact));
}

// qf == nullptr: the flags were precomputed (classify) and are not rebuilt,
// which saves reading every query record once more.
__global__ void k_init_queries(unsigned long long n, const uint8_t* kind, const double* pts,
                               uint32_t* qf, unsigned long long* toi,
                               unsigned long long* snap, unsigned long long* splits,
                               unsigned* exh_gen, uint8_t* zdiag)
{
    for (unsigned long long q = blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        toi[q] = kInfBits;
        snap[q] = kInfBits;
        splits[q] = 0;
        exh_gen[q] = kNoGen;
        zdiag[q] = 0;
        if (qf)
            qf[q] = query_flags(kind[q], pts + 24 * q);
    }
}

// Per-query outputs and the K9 reductions (global min ToI, total_splits).
// On a capacity overflow the per-query results are those folded when the
// BFS stopped (the reference returns its partial per_query, narrowphase.cpp:
// 299-302); `defaults` writes the default ToiResult instead (the seeds
// themselves exceed the capacity, narrowphase.cpp:215-218).
constexpr int kOutBlock = 256;

__global__ void __launch_bounds__(kOutBlock) k_outputs(unsigned long long n, const unsigned long long* toi,
                          const unsigned long long* splits, const unsigned* exh_gen,
                          const uint8_t* zdiag, unsigned long long max_splits,
                          NarrowScalars* sc, double* toi_out, uint8_t* flags_out, int defaults)
{
    const bool overflow = defaults != 0;
    unsigned long long mn = kInfBits, tot = 0;
    unsigned fl = 0;
    for (unsigned long long q = blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const unsigned long long tb = overflow ? kInfBits : toi[q];
        toi_out[q] = __longlong_as_double(static_cast<long long>(tb));
        const uint8_t f = overflow ? 0
                                   : static_cast<uint8_t>((exh_gen[q] != kNoGen ? CCDK_FLAG_TOLERANCE_HIT : 0u)
                                                          | (zdiag[q] ? CCDK_FLAG_ZERO_TOI_DIAG : 0u));
        flags_out[q] = f;
        fl |= f;
        mn = tb < mn ? tb : mn;
        const unsigned long long s = splits[q];
        tot += s < max_splits ? s : max_splits;
    }
    // block reduction, then one atomic of each kind per block: same-address
    // atomics from every warp serialised at L2 (~65 us per C4 launch)
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_down_sync(0xffffffffu, mn, o);
        mn = other < mn ? other : mn;
        tot += __shfl_down_sync(0xffffffffu, tot, o);
    }
    fl = __reduce_or_sync(0xffffffffu, fl);
    __shared__ unsigned long long s_mn[kOutBlock / 32], s_tot[kOutBlock / 32];
    __shared__ unsigned s_fl[kOutBlock / 32];
    const unsigned w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_mn[w] = mn;
        s_tot[w] = tot;
        s_fl[w] = fl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (unsigned i = 1; i < blockDim.x / 32; ++i) {
            mn = s_mn[i] < mn ? s_mn[i] : mn;
            tot += s_tot[i];
            fl |= s_fl[i];
        }
        atomicMin(&sc->global_toi_bits, mn);
        if (fl)
            atomicOr(&sc->any_flags, static_cast<unsigned long long>(fl));
        if (tot)
            atomicAdd(&sc->total_splits, tot);
    }
}

// ---- single-interval API kernels (inclusion_box / process_interval)

__global__ void k_inclusion(const uint8_t* kind, const double* pts, const double* boxes,
                            unsigned long long n, double* out)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    const iv::GlobalPts P { pts + 24 * i };
    const double* bx = boxes + 6 * i;
    const iv::Box b { bx[0], bx[1], bx[2], bx[3], bx[4], bx[5] };
    iv::Eval ev;
    const bool vf = kind[i] == CCDK_QUERY_VF;
    if (iv::fast_ok(P))
        iv::evaluate<iv::Fast>(vf, P, b, ev);
    else
        iv::evaluate<iv::Exact>(vf, P, b, ev);
    for (int c = 0; c < 3; ++c) {
        out[6 * i + 2 * c] = ev.range[c].lo;
        out[6 * i + 2 * c + 1] = ev.range[c].hi;
    }
}

__global__ void k_process(const uint8_t* kind, const double* pts, const double* boxes,
                          const uint16_t* depth, const double* t_star, const double* sep,
                          unsigned long long n, iv::Cfg cfg, double sep_default,
                          uint8_t* action, double* cand_t, uint8_t* zdiag, double* children,
                          uint16_t* child_depth)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    const iv::GlobalPts P { pts + 24 * i };
    const double* bx = boxes + 6 * i;
    const iv::Box b { bx[0], bx[1], bx[2], bx[3], bx[4], bx[5] };
    const double d = (sep && sep[i] >= 0.0) ? sep[i] : sep_default;
    const bool vf = kind[i] == CCDK_QUERY_VF;
    double cand = CUDART_INF;
    bool zd = false, evald = false;
    int dim = -1;
    const int act = iv::fast_ok(P)
        ? iv::process_one<iv::Fast>(vf, P, b, t_star[i], d, cfg, cand, zd, dim, evald)
        : iv::process_one<iv::Exact>(vf, P, b, t_star[i], d, cfg, cand, zd, dim, evald);
    action[i] = static_cast<uint8_t>(act);
    cand_t[i] = act == iv::kCollision ? cand : CUDART_INF;
    zdiag[i] = zd;
    // children default to a default-constructed IntervalBox ([0,1]^3, depth 0)
    double ch[12] = { 0, 1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1 };
    uint16_t cd[6] = { 0, 0, 0, 0, 0, 0 };
    if (act == iv::kSplit) {
        for (int s = 0; s < 2; ++s)
            for (int j = 0; j < 6; ++j)
                ch[6 * s + j] = bx[j];
        const double lo = bx[2 * dim], hi = bx[2 * dim + 1];
        const double mid = __dadd_rn(lo, __dmul_rn(0.5, __dsub_rn(hi, lo)));
        ch[2 * dim + 1] = mid;     // left.hi
        ch[6 + 2 * dim] = mid;     // right.lo
        for (int s = 0; s < 2; ++s)
            for (int j = 0; j < 3; ++j)
                cd[3 * s + j] = depth[3 * i + j] + (j == dim ? 1 : 0);
    }
    for (int j = 0; j < 12; ++j)
        children[12 * i + j] = ch[j];
    for (int j = 0; j < 6; ++j)
        child_depth[6 * i + j] = cd[j];
}

// ---- K7: candidate keys -> narrow queries (broadphase.cpp:194-239).
// Canonical keys list every VF pair (left = vertex) before every EE pair
// (left = edge), which is the pipeline's VF-then-EE order
// (pipeline.cpp:162-165); all pairs already passed keep_pair in the sweep.
// One warp per 32 consecutive queries: gathers in registers, then the
// warp's 32 contiguous 192-byte records (6 KiB) are written through shared
// memory as coalesced 256-byte rows; the query flags (kind | exact-widening,
// iv::kKind*) are produced here so the narrow phase need not re-read the
// records to derive them.
constexpr int kClassifyBlock = 128;

__global__ void __launch_bounds__(kClassifyBlock) k_classify_keys(
    const unsigned long long* keys, unsigned long long n, int nb, const double* __restrict__ v0,
    const double* __restrict__ v1, unsigned long long nv, const uint32_t* __restrict__ e,
    unsigned long long ne, const uint32_t* __restrict__ f, uint8_t* kind, double* pts,
    uint32_t* qflags)
{
    __shared__ double stage[kClassifyBlock / 32][32 * 24];
    const unsigned lane = threadIdx.x & 31;
    double* st = stage[threadIdx.x >> 5];
    const unsigned long long q = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    const unsigned long long q0 = q - lane; // first query of the warp
    if (q0 >= n)
        return; // warp-uniform
    if (q < n) {
        const unsigned long long key = keys[q];
        const unsigned long long lo = key >> nb;
        const unsigned long long hi = key & ((1ull << nb) - 1);
        uint32_t pv[4];
        uint8_t k;
        if (lo < nv) { // vertex-face: (p, t0, t1, t2)
            const unsigned long long fi = hi - nv - ne;
            pv[0] = static_cast<uint32_t>(lo);
            pv[1] = f[3 * fi];
            pv[2] = f[3 * fi + 1];
            pv[3] = f[3 * fi + 2];
            k = CCDK_QUERY_VF;
        } else { // edge-edge: (e0a, e0b, e1a, e1b)
            const unsigned long long ea = lo - nv, eb = hi - nv;
            pv[0] = e[2 * ea];
            pv[1] = e[2 * ea + 1];
            pv[2] = e[2 * eb];
            pv[3] = e[2 * eb + 1];
            k = CCDK_QUERY_EE;
        }
        kind[q] = k;
        bool fast = true;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double a = v0[3ull * pv[p] + c], b = v1[3ull * pv[p] + c];
                st[24 * lane + 8 * c + 2 * p] = a; // internal order (iv::GlobalPtsIL)
                st[24 * lane + 8 * c + 2 * p + 1] = b;
                fast = fast && fabs(a) <= iv::kFastLimit && fabs(b) <= iv::kFastLimit;
            }
        qflags[q] = (k == CCDK_QUERY_EE ? iv::kKindEE : 0u) | (fast ? 0u : iv::kKindExact);
    }
    __syncwarp();
    const unsigned long long valid = n - q0 < 32 ? n - q0 : 32;
    double* out = pts + 24 * q0;
    for (unsigned i = lane; i < 24 * valid; i += 32)
        out[i] = st[i];
}

// ---- K7 fused into generation 0: k_classify_keys'
// gather and coalesced record write, then each lane evaluates its query's
// root box [0,1]^3 from the coordinates still in its registers — k_gen0's
// body without re-reading the 192-byte record it just wrote (411 MB at C4).
// Generation 0's pruning snapshot is +inf and no query has split yet, so the
// root's outcome depends only on the query: bit-identical to k_gen0.
__global__ void __launch_bounds__(kClassifyBlock) k_classify_gen0(GenArgs a, ClassifySrc cs)
{
    __shared__ double stage[kClassifyBlock / 32][32 * 24];
    const unsigned lane = threadIdx.x & 31;
    double* st = stage[threadIdx.x >> 5];
    const unsigned long long q = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    const unsigned long long q0 = q - lane;
    if (q0 >= cs.n)
        return; // warp-uniform
    const bool valid = q < cs.n;
    iv::RegPts P;
    uint32_t qf = 0;
    if (valid) {
        const unsigned long long key = cs.keys[q];
        const unsigned long long lo = key >> cs.nb;
        const unsigned long long hi = key & ((1ull << cs.nb) - 1);
        uint32_t pv[4];
        uint8_t k;
        if (lo < cs.nv) { // vertex-face: (p, t0, t1, t2)
            const unsigned long long fi = hi - cs.nv - cs.ne;
            pv[0] = static_cast<uint32_t>(lo);
            pv[1] = cs.f[3 * fi];
            pv[2] = cs.f[3 * fi + 1];
            pv[3] = cs.f[3 * fi + 2];
            k = CCDK_QUERY_VF;
        } else { // edge-edge: (e0a, e0b, e1a, e1b)
            const unsigned long long ea = lo - cs.nv, eb = hi - cs.nv;
            pv[0] = cs.e[2 * ea];
            pv[1] = cs.e[2 * ea + 1];
            pv[2] = cs.e[2 * eb];
            pv[3] = cs.e[2 * eb + 1];
            k = CCDK_QUERY_EE;
        }
        cs.kind_out[q] = k;
        bool fast = true;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double x0 = cs.v0[3ull * pv[p] + c], x1 = cs.v1[3ull * pv[p] + c];
                P.x[8 * c + 2 * p] = x0;
                P.x[8 * c + 2 * p + 1] = x1;
                st[24 * lane + 8 * c + 2 * p] = x0;
                st[24 * lane + 8 * c + 2 * p + 1] = x1;
                fast = fast && fabs(x0) <= iv::kFastLimit && fabs(x1) <= iv::kFastLimit;
            }
        qf = (k == CCDK_QUERY_EE ? iv::kKindEE : 0u) | (fast ? 0u : iv::kKindExact);
        cs.qflags_out[q] = qf;
    }
    __syncwarp();
    const unsigned long long nvalid = cs.n - q0 < 32 ? cs.n - q0 : 32;
    double* out = cs.pts_out + 24 * q0;
    for (unsigned i = lane; i < 24 * nvalid; i += 32)
        out[i] = st[i];

    // generation 0 (k_gen0) on the root
    unsigned evals = 0, split_actions = 0;
    SplitRec r[2];
    r[0].dim = r[1].dim = -1;
    if (valid) {
        const iv::Box bx { 0.0, 1.0, 0.0, 1.0, 0.0, 1.0 };
        const bool vf = !(qf & iv::kKindEE);
        const double sep = a.sep ? a.sep[q] : a.sep_default;
        double cand = 0;
        bool zd = false, evald = false;
        int dim = -1, act;
        if (!(qf & iv::kKindExact)) {
            act = iv::process_one<iv::Fast, iv::RegPts, true>(vf, P, bx, CUDART_INF, sep, a.cfg, cand, zd, dim,
                                                              evald);
        } else {
            // rare (|x| > 2^1000): out of line, the register array goes by value
            const iv::Outcome o = iv::process_exact<iv::RegPts>(vf, P, bx, CUDART_INF, sep, a.cfg);
            act = o.act;
            cand = o.cand;
            zd = o.zdiag;
            dim = o.dim;
            evald = o.evaluated;
        }
        evals += evald;
        if (act == iv::kCollision) {
            record_collision(a, static_cast<unsigned>(q), cand, zd);
        } else if (act == iv::kSplit) {
            ++split_actions;
            if (!a.cfg.no_zero_toi) // a root's only request of generation 0: always admitted
                atomicAdd(&a.splits[q], 1ull);
            r[0] = { dim, 0.0, 0.0, 0.0, 0ull };
        }
    }
    append_splits(a, 1, lane, static_cast<unsigned>(valid ? q : 0), r);
    warp_add(&a.sc->evaluations, evals);
    warp_add(&a.sc->split_actions, split_actions);
}

// Reference-order query records (API input) -> internal order: (x0, x1) of
// point p, component c at 8c + 2p.
__global__ void k_records_to_internal(const double* __restrict__ ref, unsigned long long n,
                                      double* __restrict__ il)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= 24 * n)
        return;
    const unsigned long long q = i / 24;
    const int e = static_cast<int>(i - 24 * q); // reference element
    const int t = e / 12, r = e % 12;
    il[24 * q + 8 * (r % 3) + 2 * (r / 3) + t] = ref[i];
}

__global__ void k_keys_to_ids(const unsigned long long* keys, unsigned long long n, int nb,
                              const uint8_t* own_kind, const uint32_t* own_index,
                              unsigned long long nv, unsigned long long ne,
                              unsigned long long* ids, int layout)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    const unsigned long long key = keys[i];
    const unsigned long long r[2] = { key >> nb, key & ((1ull << nb) - 1) };
    for (int s = 0; s < 2; ++s) {
        unsigned long long id;
        if (own_kind) {
            id = (static_cast<unsigned long long>(own_kind[r[s]]) << 32) | own_index[r[s]];
        } else {
            const unsigned long long x = r[s];
            id = x < nv ? x : x < nv + ne ? ((1ull << 32) | (x - nv)) : ((2ull << 32) | (x - nv - ne));
        }
        if (layout == 1) // {u8 kind, 3 zero bytes, u32 index}
            id = (id >> 32) | (id << 32);
        ids[2 * i + s] = id;
    }
}

template <typename T>
T* grow(DevBuf& b, uint64_t n)
{
    return static_cast<T*>(b.ensure(n * sizeof(T)));
}

// Build (or reuse) the generation graph:
//   k_gen0 -> k_finish -> WHILE(cond) { k_generation -> k_finish }.
// The condition defaults to 1 at every launch; k_finish clears it.
void launch_generations(Ctx& c, GenArgs& a, unsigned gen0_grid, unsigned gen_grid, unsigned fin_grid,
                        const ClassifySrc* fused_classify)
{
    GenGraph& G = c.gen_graph;
    struct Key {
        GenArgs a;
        ClassifySrc cs;
        unsigned gen0_grid, gen_grid, fin_grid, fused;
    } key;
    std::memset(&key, 0, sizeof key);
    key.a = a;
    key.a.cond = 0;
    if (fused_classify)
        key.cs = *fused_classify;
    key.gen0_grid = gen0_grid;
    key.gen_grid = gen_grid;
    key.fin_grid = fin_grid;
    key.fused = fused_classify != nullptr;
    static_assert(sizeof(Key) <= sizeof(G.key), "graph key too large");
    if (G.exec && G.key_size == sizeof key && std::memcmp(G.key, &key, sizeof key) == 0) {
        CCDK_CUDA_CHECK(cudaGraphLaunch(G.exec, c.stream));
        return;
    }
    G.reset();
    CCDK_CUDA_CHECK(cudaGraphCreate(&G.graph, 0));
    cudaGraphConditionalHandle h;
    CCDK_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, G.graph, 1, cudaGraphCondAssignDefault));
    GenArgs a0 = a; // generation 0 and its finish run outside the loop
    a0.cond = 0;
    a.cond = h;
    ClassifySrc cs0 = fused_classify ? *fused_classify : ClassifySrc {};
    void* params0[] = { &a0, &cs0 };
    void* params[] = { &a };
    cudaKernelNodeParams kp {};
    if (fused_classify) { // K7 + generation 0 in one kernel
        kp.func = reinterpret_cast<void*>(k_classify_gen0);
        kp.gridDim = grid_for(fused_classify->n, kClassifyBlock);
        kp.blockDim = dim3(kClassifyBlock);
    } else {
        kp.func = reinterpret_cast<void*>(k_gen0);
        kp.gridDim = dim3(gen0_grid);
        kp.blockDim = dim3(kGenBlock);
    }
    kp.kernelParams = params0;
    cudaGraphNode_t g0, f0;
    CCDK_CUDA_CHECK(cudaGraphAddKernelNode(&g0, G.graph, nullptr, 0, &kp));
    kp.func = reinterpret_cast<void*>(k_finish);
    kp.gridDim = dim3(fin_grid);
    kp.blockDim = dim3(256);
    CCDK_CUDA_CHECK(cudaGraphAddKernelNode(&f0, G.graph, &g0, 1, &kp));
    cudaGraphNodeParams cp {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CCDK_CUDA_CHECK(cudaGraphAddNode(&cnode, G.graph, &f0, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // body: kGenUnroll x (generation kernel -> its finish), a chain; once a
    // finish clears `cont` the rest of the chain exits at once, and the
    // loop condition is the last finish's value (fewer conditional-node
    // evaluations per generation)
    // Edges inside the chain are programmatic (PDL): a kernel is launched as
    // soon as every block of its predecessor has started, and waits in
    // cudaGridDependencySynchronize() for the predecessor's completion and
    // memory, so launch latency overlaps the predecessor's tail.  Safe: the
    // predecessor's blocks are all running by then, so they finish whatever
    // the early blocks occupy.
    cudaGraphEdgeData pdl {};
    pdl.from_port = cudaGraphKernelNodePortLaunchCompletion;
    pdl.type = cudaGraphDependencyTypeProgrammatic;
    cudaGraphNode_t prev = nullptr;
    for (int u = 0; u < kGenUnroll; ++u) {
        kp.func = reinterpret_cast<void*>(k_generation);
        kp.gridDim = dim3(gen_grid);
        kp.blockDim = dim3(kGenBlock);
        kp.sharedMemBytes = kGenSmem;
        kp.kernelParams = params;
        cudaGraphNode_t gnode, fnode;
        CCDK_CUDA_CHECK(cudaGraphAddKernelNode(&gnode, body, nullptr, 0, &kp));
        if (prev)
            CCDK_CUDA_CHECK(cudaGraphAddDependencies_v2(body, &prev, &gnode, kUsePdl ? &pdl : nullptr, 1));
        kp.func = reinterpret_cast<void*>(k_finish);
        kp.gridDim = dim3(fin_grid);
        kp.blockDim = dim3(256);
        kp.sharedMemBytes = 0;
        CCDK_CUDA_CHECK(cudaGraphAddKernelNode(&fnode, body, nullptr, 0, &kp));
        CCDK_CUDA_CHECK(cudaGraphAddDependencies_v2(body, &gnode, &fnode, kUsePdl ? &pdl : nullptr, 1));
        prev = fnode;
    }
    CCDK_CUDA_CHECK(cudaGraphInstantiate(&G.exec, G.graph, 0));
    std::memcpy(G.key, &key, sizeof key);
    G.key_size = sizeof key;
    CCDK_CUDA_CHECK(cudaGraphLaunch(G.exec, c.stream));
}

// One device run over queries [0, n) of `in`; returns false on physical
// interval-buffer overflow (caller halves).
bool run_once(Ctx& c, const NarrowIn& in, uint64_t n, const uint8_t* kind, const double* pts,
              const double* sep, const uint32_t* qflags, double* toi_out, uint8_t* flags_out,
              ccdk_narrow_stats& st, uint64_t sem_cap, uint64_t gen_stop)
{
    cudaStream_t s = c.stream;
    // interval capacity per generation; stored as split records (2 intervals
    // each) in 3 regions that may each have to hold all of them
    constexpr uint64_t kBytesPerInterval = 3 * 36 / 2 * 2; // 3 regions x record / 2 x double buffer
    uint64_t cap = c.interval_capacity;
    if (cap == 0) {
        // size from free memory, probed once per query count (cudaMemGetInfo
        // is a slow driver query; keep it off the steady-state path)
        if (c.mem_probe_n == 0 || n > c.mem_probe_n) {
            size_t free_b = 0, total_b = 0;
            CCDK_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
            size_t held = 0; // already-allocated record buffers count as available
            for (int b = 0; b < 2; ++b)
                for (int d = 0; d < 3; ++d)
                    held += c.iv_qid[b][d].cap + c.iv_t[b][d].cap + c.iv_u[b][d].cap + c.iv_v[b][d].cap
                        + c.iv_dep[b][d].cap;
            c.mem_probe_cap = static_cast<uint64_t>((free_b + held) / 2) / kBytesPerInterval;
            c.mem_probe_n = n;
        }
        cap = std::max<uint64_t>(4 * n, uint64_t(1) << 24);
        cap = std::min<uint64_t>(cap, c.mem_probe_cap);
        cap = std::max<uint64_t>(cap, n);
    }
    // K7 fused into generation 0 when this run covers exactly the records the
    // pipeline left unwritten (ensure_classified writes them otherwise)
    const ClassifySrc* fused_classify = nullptr;
    if (c.classify_pending && c.classify_pending->kind_out == kind && c.classify_pending->n == n && cap >= n)
        fused_classify = c.classify_pending;
    else
        ensure_classified(c);
    if (cap < n)
        return false;
    const uint64_t cap_pairs = std::max<uint64_t>(cap / 2, 1);
    GenArgs a {};
    a.kind = kind;
    a.qf = qflags ? const_cast<uint32_t*>(qflags) : grow<uint32_t>(c.q_flags, n);
    a.pts = pts;
    a.sep = sep;
    a.sep_default = in.cfg.min_separation;
    a.cfg = { in.cfg.delta, in.cfg.t_max, in.cfg.no_zero_toi };
    a.max_splits = in.cfg.max_splits;
    a.toi = grow<unsigned long long>(c.toi_live, n);
    a.snap = grow<unsigned long long>(c.toi_snap, n);
    a.splits = grow<unsigned long long>(c.splits, n);
    a.exh_gen = grow<unsigned>(c.exh_gen, n);
    a.zdiag = grow<uint8_t>(c.zdiag, n);
    a.dirty = grow<unsigned>(c.dirty, 2 * n);
    for (int b = 0; b < 2; ++b)
        for (int d = 0; d < 3; ++d) {
            Region& R = a.reg[b][d];
            R.qid = grow<uint32_t>(c.iv_qid[b][d], cap_pairs);
            R.t = grow<double>(c.iv_t[b][d], cap_pairs);
            R.u = grow<double>(c.iv_u[b][d], cap_pairs);
            R.v = grow<double>(c.iv_v[b][d], cap_pairs);
            R.dep = grow<unsigned long long>(c.iv_dep[b][d], cap_pairs);
        }
    a.cap_pairs = cap_pairs;
    a.sem_cap = sem_cap;
    a.gen_stop = gen_stop;
    a.sc = static_cast<NarrowScalars*>(c.nscal.ensure(sizeof(NarrowScalars)));
    a.gen_sizes = grow<unsigned long long>(c.gen_sizes, kMaxGens);

    // scalars initialised by a kernel, not a host-to-device copy: the copy
    // engine serves H2D copies in order across streams, so during a chunked
    // upload a tiny copy here would wait behind all the bulk uploads
    k_init_scalars<<<1, 32, 0, s>>>(a.sc, n);
    const dim3 ig = grid_for(n, 256);
    k_init_queries<<<std::min<unsigned>(ig.x, 65535u), 256, 0, s>>>(n, kind, pts, qflags ? nullptr : a.qf,
                                                                   a.toi, a.snap, a.splits, a.exh_gen,
                                                                   a.zdiag);
    CCDK_LAUNCH_CHECK();

    if (c.gen_blocks_per_sm == 0) {
        CCDK_CUDA_CHECK(cudaFuncSetAttribute(k_generation, cudaFuncAttributeMaxDynamicSharedMemorySize, kGenSmem));
        CCDK_CUDA_CHECK(cudaFuncSetAttribute(k_generation, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        CCDK_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.gen_blocks_per_sm, k_generation, kGenBlock,
                                                                      kGenSmem));
        c.gen_blocks_per_sm = std::max(1, c.gen_blocks_per_sm);
    }
    const unsigned gen_grid = static_cast<unsigned>(c.gen_blocks_per_sm * c.num_sms);
    const unsigned gen0_grid = static_cast<unsigned>(std::min<uint64_t>((n + kGenBlock - 1) / kGenBlock,
                                                                        uint64_t(8) * c.num_sms));
    // k_finish blocks (CCDK_FIN_BLOCKS: A/B switch; default one per SM)
    static const unsigned fin_env = [] {
        const char* e = std::getenv("CCDK_FIN_BLOCKS");
        return e && *e ? static_cast<unsigned>(std::strtoul(e, nullptr, 10)) : 0u;
    }();
    const unsigned fin_grid = fin_env ? fin_env : static_cast<unsigned>(c.num_sms);

    if (c.exp && c.exp->pending)
        export_issue(c); // candidate export D2H runs under the generations
    static const bool no_graph = std::getenv("CCDK_NO_GRAPH") != nullptr;
    if (fused_classify)
        c.classify_pending = nullptr; // written by k_classify_gen0 below
    if (!no_graph) {
        launch_generations(c, a, gen0_grid, gen_grid, fin_grid, fused_classify);
    } else {
        // direct launches (profilers cannot see kernel nodes under a
        // conditional node): batches of 8 generations, then a host check
        a.cond = 0;
        NarrowScalars* hs = static_cast<NarrowScalars*>(c.pin.ensure(sizeof(NarrowScalars)));
        if (fused_classify)
            k_classify_gen0<<<grid_for(fused_classify->n, kClassifyBlock), kClassifyBlock, 0, s>>>(a, *fused_classify);
        else
            k_gen0<<<gen0_grid, kGenBlock, 0, s>>>(a);
        k_finish<<<fin_grid, 256, 0, s>>>(a);
        for (;;) {
            for (int g = 0; g < 8; ++g) {
                k_generation<<<gen_grid, kGenBlock, kGenSmem, s>>>(a);
                if (debug_enabled()) {
                    const cudaError_t e = cudaStreamSynchronize(s);
                    fprintf(stderr, "[ccdk narrow] k_generation: %s\n", cudaGetErrorString(e));
                }
                k_finish<<<fin_grid, 256, 0, s>>>(a);
                if (debug_enabled()) {
                    const cudaError_t e = cudaStreamSynchronize(s);
                    fprintf(stderr, "[ccdk narrow] k_finish: %s\n", cudaGetErrorString(e));
                }
            }
            CCDK_LAUNCH_CHECK();
            CCDK_CUDA_CHECK(cudaMemcpyAsync(hs, a.sc, sizeof(NarrowScalars), cudaMemcpyDeviceToHost, s));
            CCDK_CUDA_CHECK(cudaStreamSynchronize(s));
            if (!hs->cont)
                break;
        }
    }
    // per-query outputs right behind the generations (discarded on a
    // physical overflow, when the caller halves), then one read-back
    k_outputs<<<std::min<unsigned>(ig.x, 4 * c.num_sms), kOutBlock, 0, s>>>(n, a.toi, a.splits, a.exh_gen,
                                                              a.zdiag, a.max_splits, a.sc,
                                                              toi_out, flags_out, 0);
    CCDK_LAUNCH_CHECK();
    NarrowScalars* host_sc = static_cast<NarrowScalars*>(c.pin.ensure(sizeof(NarrowScalars)));
    CCDK_CUDA_CHECK(cudaMemcpyAsync(host_sc, a.sc, sizeof(NarrowScalars), cudaMemcpyDeviceToHost, s));
    unsigned long long* host_gs = static_cast<unsigned long long*>(c.pin_gens.ensure(kMaxGens * 8));
    CCDK_CUDA_CHECK(cudaMemcpyAsync(host_gs, a.gen_sizes, kMaxGens * 8, cudaMemcpyDeviceToHost, s));
    CCDK_CUDA_CHECK(cudaStreamSynchronize(s));
    // k_init_scalars, k_init_queries, k_gen0 + finish, the unrolled loop's
    // pairs (whole iterations), k_outputs
    c.narrow_launches += 5 + 2 * kGenUnroll * ((host_sc->gen + kGenUnroll - 2) / kGenUnroll);
#ifdef CCDK_STATS
    fprintf(stderr, "[ccdk stats] pairs with a live child %llu, with exactly one %llu\n", host_sc->vf_count,
            host_sc->next_n);
#endif
    if (debug_enabled())
        fprintf(stderr, "[ccdk narrow] n=%llu gen=%llu peak=%llu evals=%llu splits=%llu phys=%llu sem=%llu\n",
                (unsigned long long)n, host_sc->gen, host_sc->peak, host_sc->evaluations,
                host_sc->split_actions, host_sc->phys_overflow, host_sc->sem_overflow);
    if (host_sc->gen_limit)
        throw Error(CCDK_CUDA, "narrow phase: generation limit exceeded (internal error)");
    if (host_sc->phys_overflow)
        return false;
    if (host_sc->sem_overflow) // sticky across the runs of one narrow phase
        st.overflow = 1;
    const double g = __builtin_bit_cast(double, static_cast<uint64_t>(host_sc->global_toi_bits));
    st.global_toi = st.overflow ? INFINITY : std::min(st.global_toi, g);
    st.peak_queue = std::max<uint64_t>(st.peak_queue, std::max<uint64_t>(host_sc->peak, n));
    // per-generation queue sizes of independent query subsets add up: the
    // combined peak of a split run (physical halving, chunked upload) is the
    // max over generations of the sums, exactly the reference's peak_queue
    const uint64_t ng = std::min<uint64_t>(host_sc->gen, kMaxGens);
    if (c.gen_acc.size() < ng)
        c.gen_acc.resize(ng, 0);
    for (uint64_t g = 0; g < ng; ++g)
        c.gen_acc[g] += host_gs[g];
    static const bool gen_trace = std::getenv("CCDK_GEN_TRACE") != nullptr;
    if (gen_trace) { // diagnostics: intervals per generation of this run
        fprintf(stderr, "[ccdk gens] n=%llu", (unsigned long long)n);
        for (uint64_t g = 0; g < ng; ++g)
            fprintf(stderr, " %llu", (unsigned long long)host_gs[g]);
        fprintf(stderr, "\n");
    }
    st.total_splits += host_sc->total_splits;
    st.evaluations += host_sc->evaluations;
    st.split_actions += host_sc->split_actions;
    st.generations = std::max<uint64_t>(st.generations, host_sc->gen);
    c.narrow_any_flags |= host_sc->any_flags;
    return true;
}

constexpr uint64_t kNoStop = ~0ull;

// Run queries [lo, hi) to completion, halving on a physical interval-buffer
// overflow; `leaves` receives the query ranges that completed.
void run_range(Ctx& c, const NarrowIn& in, uint64_t lo, uint64_t hi, double* toi_out,
               uint8_t* flags_out, ccdk_narrow_stats& st, uint64_t sem_cap, uint64_t gen_stop,
               std::vector<std::pair<uint64_t, uint64_t>>& leaves)
{
    const uint64_t n = hi - lo;
    if (n == 0)
        return;
    if (run_once(c, in, n, in.kind + lo, in.points + 24 * lo, in.sep ? in.sep + lo : nullptr,
                 in.qflags ? in.qflags + lo : nullptr, toi_out + lo, flags_out + lo, st, sem_cap, gen_stop)) {
        leaves.emplace_back(lo, hi);
        return;
    }
    if (n <= 1)
        throw Error(CCDK_CAPACITY, "narrow phase: interval buffer cannot hold one query's frontier");
    const uint64_t mid = lo + n / 2;
    run_range(c, in, lo, mid, toi_out, flags_out, st, sem_cap, gen_stop, leaves);
    run_range(c, in, mid, hi, toi_out, flags_out, st, sem_cap, gen_stop, leaves);
}

} // namespace

void narrow_phase(Ctx& c, const NarrowIn& in, NarrowOut& out)
{
    ccdk_narrow_stats st {};
    st.global_toi = INFINITY;
    c.narrow_launches = 0;
    c.narrow_any_flags = 0;
    const uint64_t n = in.n;
    out.toi = grow<double>(c.out_toi, n);
    out.flags = grow<uint8_t>(c.out_flags, n);
    if (!c.gen_acc_keep)
        c.gen_acc.clear();
    cudaEvent_t e0 = c.events.get(EventPool::kNarrow), e1 = c.events.get(EventPool::kNarrow + 1);
    CCDK_CUDA_CHECK(cudaEventRecord(e0, c.stream));
    const bool bounded = in.queue_capacity != UINT64_MAX;
    if (n > in.queue_capacity || n == 0)
        ensure_classified(c); // no device run over these records: write them now
    if (n > 0 && n > in.queue_capacity) {
        // narrowphase.cpp:215-218: seeds alone exceed the capacity
        st.overflow = 1;
        st.peak_queue = 0;
        CCDK_CUDA_CHECK(cudaMemsetAsync(out.flags, 0, n, c.stream));
        const dim3 g = grid_for(n, 256);
        NarrowScalars* sc = static_cast<NarrowScalars*>(c.nscal.ensure(sizeof(NarrowScalars)));
        NarrowScalars init {};
        init.sem_overflow = 1;
        init.global_toi_bits = kInfBits;
        CCDK_CUDA_CHECK(cudaMemcpyAsync(sc, &init, sizeof init, cudaMemcpyHostToDevice, c.stream));
        unsigned long long* dummy = grow<unsigned long long>(c.toi_live, n);
        k_outputs<<<std::min<unsigned>(g.x, 4 * c.num_sms), kOutBlock, 0, c.stream>>>(
            n, dummy, dummy, grow<unsigned>(c.exh_gen, n), grow<uint8_t>(c.zdiag, n), 0, sc,
            out.toi, out.flags, 1);
        CCDK_LAUNCH_CHECK();
    } else if (n > 0) {
        std::vector<std::pair<uint64_t, uint64_t>> leaves;
        const std::vector<uint64_t> acc0 = c.gen_acc; // chunked callers' sums so far
        run_range(c, in, 0, n, out.toi, out.flags, st, in.queue_capacity, kNoStop, leaves);
        if (bounded && leaves.size() > 1) {
            // The batch ran as several device runs (physical halving), each
            // checked against the capacity on its own; the reference checks
            // the WHOLE batch's queue per generation (narrowphase.cpp:299-302).
            // A part's queue never exceeds the whole's, so a part overflowing
            // means the whole overflowed at the same or an earlier
            // generation.  Re-decide on the summed per-generation sizes:
            // complete them first if a part stopped early (re-run unbounded),
            // then, if some generation g's summed queue exceeds the capacity,
            // the reference stopped after generation g-1: re-run every part to
            // exactly that generation for its partial per-query results.
            auto summed = [&](size_t g) { return c.gen_acc[g] - (g < acc0.size() ? acc0[g] : 0); };
            auto rerun = [&](uint64_t gen_stop) {
                c.gen_acc = acc0;
                ccdk_narrow_stats s2 {};
                s2.global_toi = INFINITY;
                std::vector<std::pair<uint64_t, uint64_t>> refined;
                for (auto& lf : leaves)
                    run_range(c, in, lf.first, lf.second, out.toi, out.flags, s2, UINT64_MAX, gen_stop, refined);
                leaves.swap(refined);
                st = s2;
            };
            if (st.overflow)
                rerun(kNoStop);
            uint64_t first = kNoStop;
            for (size_t g = 1; g < c.gen_acc.size(); ++g)
                if (summed(g) > in.queue_capacity) {
                    first = g;
                    break;
                }
            if (first != kNoStop) {
                rerun(first - 1);
                st.overflow = 1;
            }
        }
    }
    CCDK_CUDA_CHECK(cudaEventRecord(e1, c.stream));
    CCDK_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    CCDK_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    st.device_ms = ms;
    if (n > 0 && !(n > in.queue_capacity)) {
        // narrowphase.cpp:227, 303: max over the (summed) generation queues
        st.peak_queue = 0;
        for (uint64_t v : c.gen_acc)
            st.peak_queue = std::max<uint64_t>(st.peak_queue, v);
    }
    if (st.overflow)
        st.global_toi = INFINITY; // left at kNoCollision on overflow (narrowphase.cpp:307-309)
    out.stats = st;
    out.launches = c.narrow_launches;
    out.any_flags = st.overflow ? 0 : c.narrow_any_flags;
}

void launch_inclusion(Ctx& c, const uint8_t* kind, const double* pts, const double* boxes,
                      uint64_t n, double* out)
{
    if (!n)
        return;
    k_inclusion<<<grid_for(n, 128), 128, 0, c.stream>>>(kind, pts, boxes, n, out);
    CCDK_LAUNCH_CHECK();
}

void launch_process(Ctx& c, const uint8_t* kind, const double* pts, const double* boxes,
                    const uint16_t* depth, const double* t_star, const double* sep, uint64_t n,
                    const ccdk_narrow_cfg& cfg, uint8_t* action, double* cand_t, uint8_t* zdiag,
                    double* children, uint16_t* child_depth)
{
    if (!n)
        return;
    const iv::Cfg ic { cfg.delta, cfg.t_max, cfg.no_zero_toi };
    k_process<<<grid_for(n, 128), 128, 0, c.stream>>>(kind, pts, boxes, depth, t_star, sep, n, ic,
                                                      cfg.min_separation, action, cand_t, zdiag,
                                                      children, child_depth);
    CCDK_LAUNCH_CHECK();
}

void ensure_classified(Ctx& c)
{
    if (!c.classify_pending)
        return;
    const ClassifySrc cs = *c.classify_pending;
    c.classify_pending = nullptr;
    launch_classify_keys(c, cs.keys, cs.n, cs.nb, cs.v0, cs.v1, cs.nv, cs.e, cs.ne, cs.f, cs.kind_out, cs.pts_out,
                         cs.qflags_out);
}

void launch_classify_keys(Ctx& c, const uint64_t* keys, uint64_t n, int nb, const double* v0,
                          const double* v1, uint64_t nv, const uint32_t* e, uint64_t ne,
                          const uint32_t* f, uint8_t* kind, double* pts, uint32_t* qflags)
{
    if (!n)
        return;
    k_classify_keys<<<grid_for(n, kClassifyBlock), kClassifyBlock, 0, c.stream>>>(
        reinterpret_cast<const unsigned long long*>(keys), n, nb, v0, v1, nv, e, ne, f, kind, pts, qflags);
    CCDK_LAUNCH_CHECK();
}

// Device-to-device copy by a kernel: a cudaMemcpyAsync would go through a
// copy engine and queue behind a concurrent bulk upload.
__global__ void k_copy_bytes(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                             unsigned long long bytes)
{
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long n8 = bytes / 8;
    const unsigned long long* s8 = reinterpret_cast<const unsigned long long*>(src);
    unsigned long long* d8 = reinterpret_cast<unsigned long long*>(dst);
    const bool aligned = (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 8 == 0;
    unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (aligned) {
        for (unsigned long long j = i; j < n8; j += stride)
            d8[j] = s8[j];
        for (unsigned long long j = 8 * n8 + i; j < bytes; j += stride)
            dst[j] = src[j];
    } else {
        for (unsigned long long j = i; j < bytes; j += stride)
            dst[j] = src[j];
    }
}

void launch_copy_device(Ctx& c, const void* src, void* dst, uint64_t bytes)
{
    if (!bytes)
        return;
    k_copy_bytes<<<std::min<unsigned>(grid_for(bytes / 8 + 1, 256).x, 4 * c.num_sms), 256, 0, c.stream>>>(
        static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst), bytes);
    CCDK_LAUNCH_CHECK();
}

void launch_records_to_internal(Ctx& c, const double* ref, uint64_t n, double* il)
{
    if (!n)
        return;
    k_records_to_internal<<<grid_for(24 * n, 256), 256, 0, c.stream>>>(ref, n, il);
    CCDK_LAUNCH_CHECK();
}

void launch_keys_to_ids(Ctx& c, const uint64_t* keys, uint64_t n, int nb, const uint8_t* own_kind,
                        const uint32_t* own_index, uint64_t nv, uint64_t ne, uint64_t* ids, int layout,
                        cudaStream_t stream)
{
    if (!n)
        return;
    k_keys_to_ids<<<grid_for(n, 256), 256, 0, stream ? stream : c.stream>>>(
        reinterpret_cast<const unsigned long long*>(keys), n, nb, own_kind, own_index, nv, ne,
        reinterpret_cast<unsigned long long*>(ids), layout);
    CCDK_LAUNCH_CHECK();
}

} // namespace ccdk
