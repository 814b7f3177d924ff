// Outward-rounded fp64 interval inclusion of the CCD root function, bit-exact
// with the reference (proj/include/ccdkit/interval.hpp:16-92 and
// proj/src/narrowphase.cpp:30-187).
//
// Exactness rules: every arithmetic op is an explicit
// round-to-nearest intrinsic (__dadd_rn/__dsub_rn/__dmul_rn: no FMA
// contraction whatever the flags), and every result bound moves exactly one
// representable step outward, with |x| < 1e-250 flushed to +/-1e-250.
//
// Two widening policies:
//   Fast  — nextafter as ONE directed-rounding add: x (+)_ru 2^-1074 is the
//           successor of x for every finite |x| >= 1e-250 (the exact sum lies
//           strictly between x and its successor), so up(x) is DADD.RU plus a
//           |x| < kFlush select.  Equal to the reference's bit increment for
//           every finite x; differs only for x = -inf (reference: -DBL_MAX).
//   Exact — the reference's integer bit increment incl. inf/NaN handling.
// A query whose coordinates all satisfy |x| <= 2^1000 can never produce an
// infinity inside evaluate_box (|F| <= 18 max|x| + rounding), so Fast is
// exact for it; the kernels route any other query through Exact.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <type_traits>

namespace ccdk {
namespace iv {

constexpr double kFlush = 1e-250;                   // interval.hpp:34
constexpr double kTiny = 4.9406564584124654e-324;   // 2^-1074
constexpr double kFastLimit = 1.0715086071862673e+301; // 2^1000

struct Fast {
    static __device__ __forceinline__ double up(double x)
    {
        const double r = __dadd_ru(x, kTiny);
        return fabs(x) < kFlush ? kFlush : r;
    }
    static __device__ __forceinline__ double dn(double x)
    {
        const double r = __dadd_rd(x, -kTiny);
        return fabs(x) < kFlush ? -kFlush : r;
    }
};

struct Exact {
    static __device__ __forceinline__ double up(double x)
    {
        if (isnan(x) || x == CUDART_INF)
            return x;
        if (x < kFlush && x > -kFlush)
            return kFlush;
        unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
        b += (b >> 63) ? ~0ull : 1ull; // toward +inf: +1 ulp for x >= 0, -1 for x < 0
        return __longlong_as_double(static_cast<long long>(b));
    }
    static __device__ __forceinline__ double dn(double x) { return -up(-x); }
};

struct I {
    double lo, hi;
};

template <class W>
__device__ __forceinline__ I add(I a, I b)
{
    return { W::dn(__dadd_rn(a.lo, b.lo)), W::up(__dadd_rn(a.hi, b.hi)) };
}

template <class W>
__device__ __forceinline__ I sub(I a, I b)
{
    return { W::dn(__dsub_rn(a.lo, b.hi)), W::up(__dsub_rn(a.hi, b.lo)) };
}

// scale_nn (narrowphase.cpp:30-33): exact point factor p in [0, 1].
template <class W>
__device__ __forceinline__ I scale(double p, I a)
{
    return { W::dn(__dmul_rn(p, a.lo)), W::up(__dmul_rn(p, a.hi)) };
}

// std::min / std::max semantics (first argument wins ties / NaN)
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ double mid2(I a) { return __dmul_rn(0.5, __dadd_rn(a.lo, a.hi)); }

// Width 2^-d of a dyadic domain interval at bisection depth d (d <= 1074).
__device__ __forceinline__ double dyadic_width(unsigned d)
{
    if (d <= 1022)
        return __longlong_as_double(static_cast<long long>(1023 - d) << 52);
    return __longlong_as_double(1ll << (1074 - d));
}

struct Box {
    double tlo, thi, ulo, uhi, vlo, vhi;
};

struct Eval {
    I range[3];
    double infl[3]; // influences(), narrowphase.cpp:89-107
};

// evaluate_box (narrowphase.cpp:35-85) + influences (89-107).
//
// Same operations and the same operands as the reference, reorganised so the
// live set stays small: components are independent, so the loop runs
// component-outer; point deltas are formed once per component (the reference
// forms the same values once per t-end); u- and v-terms that the reference
// recomputes per corner are formed once per (t-end, u) and (t-end, v).  All
// duplicated reference computations are deterministic, so the bits agree.
// Corner index bits follow the reference: bit0 = t, bit1 = u, bit2 = v.
// The hull starts from corner 0 like the reference; min/max of the remaining
// corners is order-independent (bounds are never +/-0 after widening, and a
// NaN operand is ignored by std::min/max unless it is the running value).
// Coordinate sources.  Query records come in two layouts:
//   reference (API) order — x0 of point p, component c at 3p + c, x1 at 12 + 3p + c
//     (NarrowQuery::points_t0/points_t1, broadphase.hpp:26-35);
//   narrow-phase internal order — (x0, x1) of point p, component c adjacent at
//     8c + 2p, so one 16-byte load brings both snapshots of a coordinate.
// pair(p, c) returns (x0, x1) of point p, component c; operator()(e) takes a
// reference-order element index.
struct GlobalPts { // reference order, global memory
    const double* __restrict__ p;
    __device__ __forceinline__ double operator()(int e) const { return __ldg(p + e); }
    __device__ __forceinline__ double2 pair(int pt, int c) const
    {
        return make_double2(__ldg(p + 3 * pt + c), __ldg(p + 12 + 3 * pt + c));
    }
};
struct GlobalPtsIL { // internal order, global memory (16-byte aligned records)
    const double* __restrict__ p;
    __device__ __forceinline__ double operator()(int e) const
    {
        const int t = e / 12, r = e % 12;
        return __ldg(p + 8 * (r % 3) + 2 * (r / 3) + t);
    }
    __device__ __forceinline__ double2 pair(int pt, int c) const
    {
        return __ldg(reinterpret_cast<const double2*>(p + 8 * c + 2 * pt));
    }
};
struct SmemPts { // internal order staged pair-major: pair k = 4c + p of lane l at [64 k + 2 l]
    const double* p; // stage + 2 * lane
    __device__ __forceinline__ double operator()(int e) const
    {
        const int t = e / 12, r = e % 12;
        return p[64 * (4 * (r % 3) + r / 3) + t];
    }
    __device__ __forceinline__ double2 pair(int pt, int c) const
    {
        return *reinterpret_cast<const double2*>(p + 64 * (4 * c + pt));
    }
};

struct RegPts { // internal order held in registers (compile-time indices only)
    double x[24];
    __device__ __forceinline__ double operator()(int e) const
    {
        const int t = e / 12, r = e % 12;
        return x[8 * (r % 3) + 2 * (r / 3) + t];
    }
    __device__ __forceinline__ double2 pair(int pt, int c) const
    {
        return make_double2(x[8 * c + 2 * pt], x[8 * c + 2 * pt + 1]);
    }
};

// One component c of evaluate_box: the hull `rng` of the 8 corners and the
// component's contribution to the three influences.
template <class W, class Pts>
__device__ __forceinline__ void component(bool vf, const Pts& P, const Box& b, int c, I& rng,
                                          double infl[3])
{
    {
        double x0[4];
        I dl[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const double2 xx = P.pair(p, c);
            x0[p] = xx.x;
            const double d = __dsub_rn(xx.y, x0[p]); // point(x1) - point(x0): both bounds
            dl[p] = { W::dn(d), W::up(d) };
        }
        double m0[4]; // corner midpoints at t = lo, indexed by (u bit) | (v bit) << 1
#pragma unroll
        for (int tb = 0; tb < 2; ++tb) {
            const double t = tb ? b.thi : b.tlo;
            I at[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const I s = scale<W>(t, dl[p]);
                at[p] = { W::dn(__dadd_rn(x0[p], s.lo)), W::up(__dadd_rn(x0[p], s.hi)) };
            }
            // VF: origin 1, u 1->2; EE: origin 2, u 0->1 (selects, not runtime indexing)
            I su[2], vt[2];
            const I a_org = vf ? at[1] : at[2];
            const I base = sub<W>(at[0], a_org);
            const I dv = sub<W>(at[3], a_org);
            if constexpr (std::is_same_v<W, Fast>) {
                // one formula for both kinds, as in component_pair (below)
                const I du = sub<W>(vf ? at[2] : at[0], at[1]);
#pragma unroll
                for (int cu = 0; cu < 2; ++cu)
                    su[cu] = sub<W>(base, scale<W>(cu ? b.uhi : b.ulo, du));
            } else {
                // Exact widening: NaN operands are possible, keep the
                // reference's add for EE (a negated NaN changes sign bits)
                const I a_uto = vf ? at[2] : at[1];
                const I a_ufr = vf ? at[1] : at[0];
                const I du = sub<W>(a_uto, a_ufr);
#pragma unroll
                for (int cu = 0; cu < 2; ++cu) {
                    const I ut = scale<W>(cu ? b.uhi : b.ulo, du);
                    su[cu] = vf ? sub<W>(base, ut) : add<W>(base, ut);
                }
            }
#pragma unroll
            for (int cv = 0; cv < 2; ++cv)
                vt[cv] = scale<W>(cv ? b.vhi : b.vlo, dv);
            double m[4];
#pragma unroll
            for (int uv = 0; uv < 4; ++uv) {
                const I f = sub<W>(su[uv & 1], vt[uv >> 1]);
                if (tb == 0 && uv == 0) {
                    rng = f;
                } else {
                    rng.lo = smin(rng.lo, f.lo);
                    rng.hi = smax(rng.hi, f.hi);
                }
                m[uv] = mid2(f);
            }
            // u influence: corners differing in bit1; v influence: bit2
            infl[1] = smax(infl[1], fabs(__dsub_rn(m[1], m[0])));
            infl[1] = smax(infl[1], fabs(__dsub_rn(m[3], m[2])));
            infl[2] = smax(infl[2], fabs(__dsub_rn(m[2], m[0])));
            infl[2] = smax(infl[2], fabs(__dsub_rn(m[3], m[1])));
            if (tb == 0) {
#pragma unroll
                for (int uv = 0; uv < 4; ++uv)
                    m0[uv] = m[uv];
            } else {
#pragma unroll
                for (int uv = 0; uv < 4; ++uv)
                    infl[0] = smax(infl[0], fabs(__dsub_rn(m[uv], m0[uv])));
            }
        }
    }
}

template <class W, class Pts>
__device__ __forceinline__ void evaluate(bool vf, const Pts& P, const Box& b, Eval& ev)
{
    ev.infl[0] = ev.infl[1] = ev.infl[2] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
        component<W, Pts>(vf, P, b, c, ev.range[c], ev.infl);
}

// splittable (narrowphase.cpp:109-113)
__device__ __forceinline__ bool splittable(double lo, double hi)
{
    const double mid = __dadd_rn(lo, __dmul_rn(0.5, __dsub_rn(hi, lo)));
    return mid > lo && mid < hi;
}

struct Cfg {
    double delta, t_max;
    int no_zero_toi;
};

enum : int { kPruned = 0, kCollision = 1, kSplit = 2 };

// process_interval (narrowphase.cpp:134-187).  Returns the action; for Split
// `dim` is the bisection dimension (0 t, 1 u, 2 v).
template <class W, class Pts, bool kUnrollC = false>
__device__ __forceinline__ int process_one(bool vf, const Pts& P, const Box& b,
                                           double t_star, double d, const Cfg& cfg,
                                           double& cand_t, bool& zdiag, int& dim,
                                           bool& evaluated)
{
    zdiag = false;
    evaluated = false;
    dim = -1;
    if (b.tlo >= t_star || b.tlo >= cfg.t_max)
        return kPruned;
    if (vf && __dadd_rn(b.ulo, b.vlo) > 1.0)
        return kPruned;
    // Components one at a time.  A component whose range misses the
    // tolerance cube prunes the box whatever the others hold, so the loop
    // exits early; otherwise the inside test, max width and influences are
    // reduced on the fly (all order-independent).  The loop stays rolled (a
    // third of the code, so a hot loop stays in the instruction cache) unless
    // kUnrollC: coordinates held in a register array need compile-time
    // component indices.
    Eval ev;
    ev.infl[0] = ev.infl[1] = ev.infl[2] = 0.0;
    evaluated = true;
    bool inside = true;
    double wmax = 0.0;
    auto comp = [&](int c) -> bool { // true: the component prunes the box
        I rng;
        component<W, Pts>(vf, P, b, c, rng, ev.infl);
        if (rng.lo > d || rng.hi < -d)
            return true;
        inside = inside && rng.lo >= -d && rng.hi <= d;
        const double w = __dsub_rn(rng.hi, rng.lo);
        wmax = c == 0 ? w : smax(wmax, w);
        return false;
    };
    if constexpr (kUnrollC) {
        if (comp(0) || comp(1) || comp(2))
            return kPruned;
    } else {
#pragma unroll 1
        for (int c = 0; c < 3; ++c)
            if (comp(c))
                return kPruned;
    }
    const bool force_zero = cfg.no_zero_toi && b.tlo == 0.0;
    if (!force_zero) {
        if (wmax < cfg.delta || inside) {
            cand_t = b.tlo;
            return kCollision;
        }
    }
    // first splittable dimension with strictly larger influence (t < u < v
    // on ties); written without runtime array indexing to stay in registers
    double best = 0.0;
    if (splittable(b.tlo, b.thi)) {
        dim = 0;
        best = ev.infl[0];
    }
    if (splittable(b.ulo, b.uhi) && (dim < 0 || ev.infl[1] > best)) {
        dim = 1;
        best = ev.infl[1];
    }
    if (splittable(b.vlo, b.vhi) && (dim < 0 || ev.infl[2] > best))
        dim = 2;
    if (dim < 0) {
        cand_t = b.tlo;
        zdiag = force_zero;
        return kCollision;
    }
    return kSplit;
}

// ---------------------------------------------------------------- pairs
// The two children of a split along dimension D are evaluated together: they
// share the parent's samples in the other two dimensions and the midpoint in
// D, so the corner values F(t, u, v) on the shared face (and, for a u- or
// v-split, every point position P(t) and the base/du/dv terms) are formed
// once.  Every corner value is produced by exactly the operations of
// evaluate_box (narrowphase.cpp:35-85) on exactly the same operands, so each
// child's hull and influences are bit-identical to evaluating it alone; the
// hull folds a child's corners starting from its corner 0 like the
// reference, and in the Fast path (no NaN) min/max are order-independent.
// Samples: dim D holds (lo, mid, hi), the others (lo, hi); child 0 takes
// indices {0, 1} along D, child 1 {1, 2}.
#ifndef CCDK_TWICE_MID
#define CCDK_TWICE_MID 1
#endif
#ifndef CCDK_SLICE_HULL
#define CCDK_SLICE_HULL 1
#endif
#ifndef CCDK_UNIFIED_SU
#define CCDK_UNIFIED_SU 1
#endif
struct PairBox {
    double t[3], u[3], v[3];
};

// Corner "midpoints" for the influences.  With CCDK_TWICE_MID the factor 0.5
// is dropped: every influence comes out exactly twice the reference's and
// only their order is ever used (strict comparisons between the three
// dimensions, narrowphase.cpp:169-177).  Exact on the Fast path: lo + hi is 0
// or a multiple of ulp(1e-250) (|bounds| >= 1e-250 after widening), so
// neither the halving nor the halved differences can be subnormal, and
// rn((a - b) / 2) = rn(a - b) / 2 without underflow; |sums| <= 2^1007.
__device__ __forceinline__ double pair_mid(I f)
{
#if CCDK_TWICE_MID
    return __dadd_rn(f.lo, f.hi);
#else
    return mid2(f);
#endif
}

template <int D, class Pts>
__device__ __forceinline__ void component_pair(bool vf, const Pts& P, const PairBox& b, int c, I rng[2],
                                               double infl[2][3])
{
    using W = Fast;
    constexpr int NT = D == 0 ? 3 : 2, NU = D == 1 ? 3 : 2, NV = D == 2 ? 3 : 2;
    double x0[4];
    I dl[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const double2 xx = P.pair(p, c);
        x0[p] = xx.x;
        const double d = __dsub_rn(xx.y, x0[p]);
        dl[p] = { W::dn(d), W::up(d) };
    }
    double mp[NU * NV]; // corner midpoints at the previous t sample
#pragma unroll
    for (int it = 0; it < NT; ++it) {
        const double t = b.t[it];
        I at[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const I s = scale<W>(t, dl[p]);
            at[p] = { W::dn(__dadd_rn(x0[p], s.lo)), W::up(__dadd_rn(x0[p], s.hi)) };
        }
#if CCDK_UNIFIED_SU
        // One formula for both kinds (no per-lane select between add and
        // sub: predication issued both).  EE's base + u (p1 - p0) is formed
        // as base - u (p0 - p1): Fast widening is sign-symmetric
        // (dn(-x) = -up(x)) and negation is exact, so sub(p0, p1) is exactly
        // the negated sub(p1, p0), scale(u >= 0, .) commutes with it, and
        // sub(base, -w) is bit for bit add(base, w) (x - (-y) == x + y in
        // IEEE arithmetic, zeros included; the Fast path never sees a NaN).
        const I a_org = vf ? at[1] : at[2];
        const I a_uto = vf ? at[2] : at[0];
        const I base = sub<W>(at[0], a_org);
        const I du = sub<W>(a_uto, at[1]);
        const I dv = sub<W>(at[3], a_org);
        I su[NU], vt[NV];
#pragma unroll
        for (int iu = 0; iu < NU; ++iu)
            su[iu] = sub<W>(base, scale<W>(b.u[iu], du));
#else
        const I a_org = vf ? at[1] : at[2];
        const I a_uto = vf ? at[2] : at[1];
        const I a_ufr = vf ? at[1] : at[0];
        const I base = sub<W>(at[0], a_org);
        const I du = sub<W>(a_uto, a_ufr);
        const I dv = sub<W>(at[3], a_org);
        I su[NU], vt[NV];
#pragma unroll
        for (int iu = 0; iu < NU; ++iu) {
            const I ut = scale<W>(b.u[iu], du);
            su[iu] = vf ? sub<W>(base, ut) : add<W>(base, ut);
        }
#endif
#pragma unroll
        for (int iv = 0; iv < NV; ++iv)
            vt[iv] = scale<W>(b.v[iv], dv);
        double m[NU * NV];
#if CCDK_SLICE_HULL
        // Hulls through slices: the corners of one sample along D form a
        // slice whose hull is folded once and shared by both children (the
        // midpoint slice belongs to both).  min/max over a child's corners
        // is order-independent here (Fast path: no NaN; widened bounds are
        // never +/-0), so the grouping is bit-identical to the corner fold.
        auto corner = [&](int iu, int iv) -> I {
            const I f = sub<W>(su[iu], vt[iv]);
            m[iu * NV + iv] = pair_mid(f);
            return f;
        };
        auto hull = [](I& acc, const I& f) {
            acc.lo = smin(acc.lo, f.lo);
            acc.hi = smax(acc.hi, f.hi);
        };
        if constexpr (D == 0) {
            I sl = corner(0, 0);
            hull(sl, corner(0, 1));
            hull(sl, corner(1, 0));
            hull(sl, corner(1, 1));
            if (it == 0) {
                rng[0] = sl;
            } else if (it == 1) {
                hull(rng[0], sl);
                rng[1] = sl;
            } else {
                hull(rng[1], sl);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) { // sample index along D
                I sl;
                if constexpr (D == 1) {
                    sl = corner(k, 0);
                    hull(sl, corner(k, 1));
                } else {
                    sl = corner(0, k);
                    hull(sl, corner(1, k));
                }
                if (k <= 1) {
                    if (it == 0 && k == 0)
                        rng[0] = sl;
                    else
                        hull(rng[0], sl);
                }
                if (k >= 1) {
                    if (it == 0 && k == 1)
                        rng[1] = sl;
                    else
                        hull(rng[1], sl);
                }
            }
        }
#else
#pragma unroll
        for (int iu = 0; iu < NU; ++iu) {
#pragma unroll
            for (int iv = 0; iv < NV; ++iv) {
                const I f = sub<W>(su[iu], vt[iv]);
                m[iu * NV + iv] = mid2(f);
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    const int kd = D == 0 ? it : D == 1 ? iu : iv; // index along D
                    if (kd == ch || kd == ch + 1) {
                        const bool first = (D == 0 ? it == ch : it == 0) && (D == 1 ? iu == ch : iu == 0)
                            && (D == 2 ? iv == ch : iv == 0);
                        if (first) {
                            rng[ch] = f;
                        } else {
                            rng[ch].lo = smin(rng[ch].lo, f.lo);
                            rng[ch].hi = smax(rng[ch].hi, f.hi);
                        }
                    }
                }
            }
        }
#endif
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
            if (D == 0 && !(it == ch || it == ch + 1))
                continue;
            const int u0 = D == 1 ? ch : 0, v0 = D == 2 ? ch : 0;
            // u influence: corner pairs differing in u (narrowphase.cpp:89-107)
#pragma unroll
            for (int iv = v0; iv < v0 + 2; ++iv)
                infl[ch][1] = smax(infl[ch][1], fabs(__dsub_rn(m[(u0 + 1) * NV + iv], m[u0 * NV + iv])));
            // v influence
#pragma unroll
            for (int iu = u0; iu < u0 + 2; ++iu)
                infl[ch][2] = smax(infl[ch][2], fabs(__dsub_rn(m[iu * NV + v0 + 1], m[iu * NV + v0])));
            // t influence: this t sample against the previous one
            const bool tpair = D == 0 ? it == ch + 1 : it == 1;
            if (tpair) {
#pragma unroll
                for (int iu = u0; iu < u0 + 2; ++iu)
#pragma unroll
                    for (int iv = v0; iv < v0 + 2; ++iv)
                        infl[ch][0] = smax(infl[ch][0], fabs(__dsub_rn(m[iu * NV + iv], mp[iu * NV + iv])));
            }
        }
#pragma unroll
        for (int k = 0; k < NU * NV; ++k)
            mp[k] = m[k];
    }
}

struct PairOutcome {
    double cand[2];
    int act[2], dim[2];
    bool zdiag[2], evaluated[2];
};

// process_interval (narrowphase.cpp:134-187) on both children of a pair
// (Fast widening only).  `alive[ch]` is false for a child the caller has
// already pruned by t >= t*, t >= t_max or the VF simplex test.
template <int D, class Pts>
__device__ __forceinline__ PairOutcome process_pair(bool vf, const Pts& P, const PairBox& b, const bool alive0[2],
                                                    double d, const Cfg& cfg)
{
    PairOutcome o;
    bool alive[2] = { alive0[0], alive0[1] };
    bool inside[2] = { true, true };
    double wmax[2] = { 0.0, 0.0 };
    double infl[2][3] = { { 0.0, 0.0, 0.0 }, { 0.0, 0.0, 0.0 } };
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
        o.act[ch] = kPruned;
        o.dim[ch] = -1;
        o.zdiag[ch] = false;
        o.evaluated[ch] = alive[ch];
        o.cand[ch] = 0.0;
    }
#pragma unroll 1
    for (int c = 0; c < 3; ++c) {
        I rng[2];
        component_pair<D, Pts>(vf, P, b, c, rng, infl);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
            if (rng[ch].lo > d || rng[ch].hi < -d)
                alive[ch] = false;
            inside[ch] = inside[ch] && rng[ch].lo >= -d && rng[ch].hi <= d;
            // widths are >= +0 here (no NaN, hi >= lo), so folding from the
            // initial 0.0 equals starting at component 0 without a select
            wmax[ch] = smax(wmax[ch], __dsub_rn(rng[ch].hi, rng[ch].lo));
        }
        if (!alive[0] && !alive[1])
            return o;
    }
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
        if (!alive[ch])
            continue;
        const double tlo = b.t[D == 0 ? ch : 0], thi = b.t[D == 0 ? ch + 1 : 1];
        const double ulo = b.u[D == 1 ? ch : 0], uhi = b.u[D == 1 ? ch + 1 : 1];
        const double vlo = b.v[D == 2 ? ch : 0], vhi = b.v[D == 2 ? ch + 1 : 1];
        const bool force_zero = cfg.no_zero_toi && tlo == 0.0;
        if (!force_zero && (wmax[ch] < cfg.delta || inside[ch])) {
            o.cand[ch] = tlo;
            o.act[ch] = kCollision;
            continue;
        }
        int dim = -1;
        double best = 0.0;
        if (splittable(tlo, thi)) {
            dim = 0;
            best = infl[ch][0];
        }
        if (splittable(ulo, uhi) && (dim < 0 || infl[ch][1] > best)) {
            dim = 1;
            best = infl[ch][1];
        }
        if (splittable(vlo, vhi) && (dim < 0 || infl[ch][2] > best))
            dim = 2;
        if (dim < 0) {
            o.cand[ch] = tlo;
            o.zdiag[ch] = force_zero;
            o.act[ch] = kCollision;
        } else {
            o.dim[ch] = dim;
            o.act[ch] = kSplit;
        }
    }
    return o;
}

// A query takes the Fast widening when every coordinate is <= 2^1000 in
// magnitude (see the header comment).
// The Exact-widening instantiation is out of line: it runs only for queries
// beyond 2^1000 and would otherwise double the hot loop's code size.
struct Outcome {
    double cand;
    int act, dim;
    bool zdiag, evaluated;
};

template <class Pts>
__device__ __noinline__ Outcome process_exact(bool vf, const Pts P, const Box b, double t_star,
                                              double d, const Cfg cfg)
{
    Outcome o;
    o.cand = 0.0;
    o.act = process_one<Exact, Pts>(vf, P, b, t_star, d, cfg, o.cand, o.zdiag, o.dim, o.evaluated);
    return o;
}

template <class Pts>
__device__ __forceinline__ bool fast_ok(const Pts& P)
{
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 24; ++i)
        ok = ok && fabs(P(i)) <= kFastLimit; // NaN compares false -> Exact
    return ok;
}

// Query kind byte as stored on the device: bit0 = edge-edge, bit1 = the query
// needs the Exact widening (set once per narrow phase by the init kernel).
constexpr uint8_t kKindEE = 1, kKindExact = 2;

} // namespace iv
} // namespace ccdk
