// K1: swept-AABB build (proj/src/aabb.cpp:10-112).
//
// One thread per primitive slot (V, then E, then F, each in index order:
// aabb.cpp:79-105).  Extents are fp64 min/max over both snapshots with
// std::min/max semantics, inflation is `pad = inflation*(hi-lo)` with the
// 1e-12 floor (aabb.cpp:51-58, aabb.hpp:44), and the outward fp64 -> fp32
// rounding is the directed conversion cvt.rm/.rp (F2F.F32.F64.RM/RP): for
// every finite x it equals round_down/up_reduced (largest float <= x /
// smallest float >= x, incl. overflow to +/-FLT_MAX/inf and subnormals, no FTZ).
//
// Outputs are SoA per axis (bmin[axis*k + s]) for coalesced sweep staging,
// plus the owner's mesh-vertex triple (absent = 0xffffffff) and its rank.
#include <math_constants.h>

#include "ccdk_internal.cuh"

namespace ccdk {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

__global__ void k_round(const double* x, unsigned long long n, float* dn, float* up,
                        unsigned long long* err)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    const double v = x[i];
    if (!isfinite(v)) {
        atomicMin(err, i); // round_*_reduced throw InvalidInput (aabb.cpp:12-13)
        return;
    }
    dn[i] = __double2float_rd(v);
    up[i] = __double2float_ru(v);
}

__global__ void __launch_bounds__(256) k_build_boxes(
    const double* __restrict__ v0, const double* __restrict__ v1, unsigned long long nv,
    const uint32_t* __restrict__ e, unsigned long long ne, const uint32_t* __restrict__ f,
    unsigned long long nf, double inflation, float* __restrict__ bmin, float* __restrict__ bmax,
    uint4* __restrict__ vids, unsigned long long* err)
{
    const unsigned long long k = nv + ne + nf;
    const unsigned long long s = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (s >= k)
        return;
    uint32_t w[3] = { kNone, kNone, kNone };
    int nw;
    if (s < nv) {
        w[0] = static_cast<uint32_t>(s);
        nw = 1;
    } else if (s < nv + ne) {
        const unsigned long long i = s - nv;
        w[0] = e[2 * i];
        w[1] = e[2 * i + 1];
        nw = 2;
    } else {
        const unsigned long long i = s - nv - ne;
        w[0] = f[3 * i];
        w[1] = f[3 * i + 1];
        w[2] = f[3 * i + 2];
        nw = 3;
    }
    double lo[3] = { CUDART_INF, CUDART_INF, CUDART_INF };
    double hi[3] = { -CUDART_INF, -CUDART_INF, -CUDART_INF };
    for (int t = 0; t < nw; ++t) {
        const double* a = v0 + 3ull * w[t];
        const double* b = v1 + 3ull * w[t];
#pragma unroll
        for (int c = 0; c < 3; ++c) { // Extent::absorb(t0) then absorb(t1)
            const double x = a[c], y = b[c];
            lo[c] = smin(lo[c], x);
            hi[c] = smax(hi[c], x);
            lo[c] = smin(lo[c], y);
            hi[c] = smax(hi[c], y);
        }
    }
    bool bad = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double l = lo[c], h = hi[c];
        if (inflation > 0.0) {
            double pad = __dmul_rn(inflation, __dsub_rn(h, l));
            if (pad == 0.0)
                pad = 1e-12; // kZeroExtentInflation
            l = __dsub_rn(l, pad);
            h = __dadd_rn(h, pad);
        }
        bad = bad || !isfinite(l) || !isfinite(h);
        bmin[c * k + s] = __double2float_rd(l);
        bmax[c * k + s] = __double2float_ru(h);
    }
    if (bad)
        atomicMin(err, s);
    vids[s] = make_uint4(w[0], w[1], w[2], static_cast<uint32_t>(s));
}

__global__ void k_soa_to_aos(const float* bmin, const float* bmax, unsigned long long k,
                             unsigned long long nv, unsigned long long ne, float* mn, float* mx,
                             uint8_t* kind, uint32_t* index)
{
    const unsigned long long s = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (s >= k)
        return;
    for (int c = 0; c < 3; ++c) {
        mn[3 * s + c] = bmin[c * k + s];
        mx[3 * s + c] = bmax[c * k + s];
    }
    if (s < nv) {
        kind[s] = CCDK_KIND_VERTEX;
        index[s] = static_cast<uint32_t>(s);
    } else if (s < nv + ne) {
        kind[s] = CCDK_KIND_EDGE;
        index[s] = static_cast<uint32_t>(s - nv);
    } else {
        kind[s] = CCDK_KIND_FACE;
        index[s] = static_cast<uint32_t>(s - nv - ne);
    }
}

} // namespace

void launch_round(Ctx& c, const double* x, uint64_t n, float* dn, float* up)
{
    if (!n)
        return;
    auto* ctr = static_cast<DevCounters*>(c.counters.ensure(sizeof(DevCounters)));
    CCDK_CUDA_CHECK(cudaMemsetAsync(&ctr->error, 0xff, sizeof(unsigned long long), c.stream));
    k_round<<<grid_for(n, 256), 256, 0, c.stream>>>(x, n, dn, up, &ctr->error);
    CCDK_LAUNCH_CHECK();
    unsigned long long err = 0;
    CCDK_CUDA_CHECK(cudaMemcpyAsync(&err, &ctr->error, sizeof err, cudaMemcpyDeviceToHost, c.stream));
    CCDK_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (err != ~0ull)
        throw Error(CCDK_INVALID_INPUT, "round_down_reduced: non-finite input");
}

void launch_build_boxes(Ctx& c, const double* v0, const double* v1, uint64_t nv,
                        const uint32_t* e, uint64_t ne, const uint32_t* f, uint64_t nf,
                        double inflation, float* bmin, float* bmax, uint4* vids)
{
    const uint64_t k = nv + ne + nf;
    if (!k)
        return;
    auto* ctr = static_cast<DevCounters*>(c.counters.ensure(sizeof(DevCounters)));
    CCDK_CUDA_CHECK(cudaMemsetAsync(&ctr->error, 0xff, sizeof(unsigned long long), c.stream));
    k_build_boxes<<<grid_for(k, 256), 256, 0, c.stream>>>(v0, v1, nv, e, ne, f, nf, inflation,
                                                          bmin, bmax, vids, &ctr->error);
    CCDK_LAUNCH_CHECK();
}

void launch_soa_to_aos(Ctx& c, const float* bmin, const float* bmax, uint64_t k, float* mn,
                       float* mx, uint8_t* kind, uint32_t* index, uint64_t nv, uint64_t ne)
{
    if (!k)
        return;
    k_soa_to_aos<<<grid_for(k, 256), 256, 0, c.stream>>>(bmin, bmax, k, nv, ne, mn, mx, kind, index);
    CCDK_LAUNCH_CHECK();
}

} // namespace ccdk
