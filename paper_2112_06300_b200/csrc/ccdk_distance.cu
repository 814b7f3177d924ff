// Per-query minimum separations (pipeline.cpp:39-55) with the t = 0
// primitive distances of proj/src/distance.cpp:10-113, one thread per query.
//
// Same operation order as the reference (Vec3 ops and dot products left to
// right), explicit round-to-nearest intrinsics (no FMA contraction), IEEE
// sqrt and division, std::clamp / std::min semantics, so the separations are
// bit-identical.
#include "ccdk_internal.cuh"

namespace ccdk {

namespace {

struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return { __dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z) }; }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return { __dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z) }; }
__device__ __forceinline__ V3 vscale(double s, V3 v) { return { __dmul_rn(s, v.x), __dmul_rn(s, v.y), __dmul_rn(s, v.z) }; }
__device__ __forceinline__ double vdot(V3 a, V3 b)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ double sqn(V3 v) { return vdot(v, v); }
__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v); }
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }

// closest_on_segment (distance.cpp:10-19)
__device__ V3 closest_on_segment(V3 p, V3 a, V3 b)
{
    const V3 ab = vsub(b, a);
    const double len2 = sqn(ab);
    if (len2 == 0.0)
        return a;
    double t = __ddiv_rn(vdot(vsub(p, a), ab), len2);
    t = clamp01(t);
    return vadd(a, vscale(t, ab));
}

// point_triangle_distance (distance.cpp:23-75): Voronoi-region walk.
__device__ double point_triangle(V3 p, V3 a, V3 b, V3 c)
{
    const V3 ab = vsub(b, a), ac = vsub(c, a), ap = vsub(p, a);
    const double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0)
        return __dsqrt_rn(sqn(vsub(p, a)));
    const V3 bp = vsub(p, b);
    const double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3)
        return __dsqrt_rn(sqn(vsub(p, b)));
    const double vc = __dsub_rn(__dmul_rn(d1, d4), __dmul_rn(d3, d2));
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double v = __ddiv_rn(d1, __dsub_rn(d1, d3));
        return __dsqrt_rn(sqn(vsub(p, vadd(a, vscale(v, ab)))));
    }
    const V3 cp = vsub(p, c);
    const double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6)
        return __dsqrt_rn(sqn(vsub(p, c)));
    const double vb = __dsub_rn(__dmul_rn(d5, d2), __dmul_rn(d1, d6));
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = __ddiv_rn(d2, __dsub_rn(d2, d6));
        return __dsqrt_rn(sqn(vsub(p, vadd(a, vscale(w, ac)))));
    }
    const double va = __dsub_rn(__dmul_rn(d3, d6), __dmul_rn(d5, d4));
    const double e43 = __dsub_rn(d4, d3), e56 = __dsub_rn(d5, d6);
    if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {
        const double w = __ddiv_rn(e43, __dadd_rn(e43, e56));
        return __dsqrt_rn(sqn(vsub(p, vadd(b, vscale(w, vsub(c, b))))));
    }
    const double denom = __dadd_rn(__dadd_rn(va, vb), vc);
    if (denom <= 0.0) { // degenerate triangle: closest edge
        const double da = sqn(vsub(p, closest_on_segment(p, a, b)));
        const double db = sqn(vsub(p, closest_on_segment(p, b, c)));
        const double dc = sqn(vsub(p, closest_on_segment(p, c, a)));
        return __dsqrt_rn(dmin(dmin(da, db), dc));
    }
    const double v = __ddiv_rn(vb, denom), w = __ddiv_rn(vc, denom);
    return __dsqrt_rn(sqn(vsub(p, vadd(vadd(a, vscale(v, ab)), vscale(w, ac)))));
}

// segment_segment_distance (distance.cpp:77-113)
__device__ double segment_segment(V3 p0, V3 p1, V3 q0, V3 q1)
{
    const V3 d1 = vsub(p1, p0), d2 = vsub(q1, q0), r = vsub(p0, q0);
    const double a = sqn(d1), e = sqn(d2), f = vdot(d2, r);
    double s = 0.0, t = 0.0;
    if (a == 0.0 && e == 0.0) {
    } else if (a == 0.0) {
        t = clamp01(__ddiv_rn(f, e));
    } else {
        const double c = vdot(d1, r);
        if (e == 0.0) {
            s = clamp01(__ddiv_rn(-c, a));
        } else {
            const double b = vdot(d1, d2);
            const double denom = __dsub_rn(__dmul_rn(a, e), __dmul_rn(b, b));
            s = denom != 0.0 ? clamp01(__ddiv_rn(__dsub_rn(__dmul_rn(b, f), __dmul_rn(c, e)), denom)) : 0.0;
            t = __ddiv_rn(__dadd_rn(__dmul_rn(b, s), f), e);
            if (t < 0.0) {
                t = 0.0;
                s = clamp01(__ddiv_rn(-c, a));
            } else if (t > 1.0) {
                t = 1.0;
                s = clamp01(__ddiv_rn(__dsub_rn(b, c), a));
            }
        }
    }
    const V3 cp = vadd(p0, vscale(s, d1));
    const V3 cq = vadd(q0, vscale(t, d2));
    return __dsqrt_rn(sqn(vsub(cp, cq)));
}

template <bool IL>
__global__ void k_min_seps(const uint8_t* kind, const double* pts, unsigned long long n,
                           double fraction, int relative, double absolute, double* out)
{
    const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    if (!relative) {
        out[i] = absolute;
        return;
    }
    const double* R = pts + 24 * i; // t = 0 snapshot
    // element 3p + c of the t = 0 snapshot in either record order
    auto P = [&](int e) { return IL ? R[8 * (e % 3) + 2 * (e / 3)] : R[e]; };
    const V3 a { P(0), P(1), P(2) }, b { P(3), P(4), P(5) }, c { P(6), P(7), P(8) },
        d { P(9), P(10), P(11) };
    const double d0 = kind[i] == CCDK_QUERY_EE ? segment_segment(a, b, c, d) : point_triangle(a, b, c, d);
    out[i] = __dmul_rn(fraction, d0);
}

} // namespace

void launch_min_seps(Ctx& c, const uint8_t* kind, const double* pts, uint64_t n,
                     const ccdk_pipeline_cfg& cfg, double* out, bool internal)
{
    if (!n)
        return;
    auto k = internal ? k_min_seps<true> : k_min_seps<false>;
    k<<<grid_for(n, 128), 128, 0, c.stream>>>(kind, pts, n, cfg.min_sep_fraction,
                                              cfg.min_sep_mode == CCDK_MINSEP_RELATIVE,
                                              cfg.narrow.min_separation, out);
    CCDK_LAUNCH_CHECK();
}

} // namespace ccdk
