/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference ccdkit hot path
 * (see ccd_oracle.h).  Paths below are relative to /root/reference/proj/.
 *
 * Written as an independent restatement: widening uses libm nextafter rather
 * than the reference's bit increment, the broad phase is a sorted sweep with
 * run-length statistics rather than a queue, and the narrow phase keeps the
 * reference's generation/snapshot/fold semantics with a plain serial queue.
 */
#include "ccd_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

void orc_free(void* p) { free(p); }

/* ---------------------------------------------------------------- rounding */

/* aabb.cpp:10-18 — largest float <= x. */
float orc_round_down_reduced(double x)
{
    float r = (float)x;
    if ((double)r > x)
        r = nextafterf(r, -INFINITY);
    return r;
}

/* aabb.cpp:20-28 — smallest float >= x. */
float orc_round_up_reduced(double x)
{
    float r = (float)x;
    if ((double)r < x)
        r = nextafterf(r, INFINITY);
    return r;
}

/* ------------------------------------------------------------- scene checks */

/* SceneStep::validate, scene.cpp:13-34. */
static int validate_scene(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                          uint64_t ne, const uint32_t* f, uint64_t nf)
{
    for (uint64_t i = 0; i < 3 * nv; ++i)
        if (!isfinite(v0[i]) || !isfinite(v1[i]))
            return CCDK_INVALID_INPUT;
    for (uint64_t i = 0; i < ne; ++i) {
        if (e[2 * i] >= nv || e[2 * i + 1] >= nv || e[2 * i] == e[2 * i + 1])
            return CCDK_INVALID_INPUT;
    }
    for (uint64_t i = 0; i < nf; ++i) {
        const uint32_t a = f[3 * i], b = f[3 * i + 1], c = f[3 * i + 2];
        if (a >= nv || b >= nv || c >= nv || a == b || b == c || a == c)
            return CCDK_INVALID_INPUT;
    }
    return 0;
}

/* ------------------------------------------------------------------- boxes */

/* build_boxes / Extent / finish_box, aabb.cpp:32-112 (kZeroExtentInflation,
 * aabb.hpp:44).  Slot order V, E, F by index. */
int orc_build_boxes(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                    uint64_t ne, const uint32_t* f, uint64_t nf, double inflation,
                    float* mn, float* mx, uint8_t* kind, uint32_t* index)
{
    if (validate_scene(v0, v1, nv, e, ne, f, nf))
        return CCDK_INVALID_INPUT;
    if (inflation < 0.0)
        return CCDK_INVALID_INPUT;
    const uint64_t k = nv + ne + nf;
    for (uint64_t s = 0; s < k; ++s) {
        uint32_t verts[3];
        int nverts;
        if (s < nv) {
            kind[s] = CCDK_KIND_VERTEX;
            index[s] = (uint32_t)s;
            verts[0] = (uint32_t)s;
            nverts = 1;
        } else if (s < nv + ne) {
            const uint64_t i = s - nv;
            kind[s] = CCDK_KIND_EDGE;
            index[s] = (uint32_t)i;
            verts[0] = e[2 * i];
            verts[1] = e[2 * i + 1];
            nverts = 2;
        } else {
            const uint64_t i = s - nv - ne;
            kind[s] = CCDK_KIND_FACE;
            index[s] = (uint32_t)i;
            verts[0] = f[3 * i];
            verts[1] = f[3 * i + 1];
            verts[2] = f[3 * i + 2];
            nverts = 3;
        }
        for (int c = 0; c < 3; ++c) {
            double lo = INFINITY, hi = -INFINITY;
            for (int t = 0; t < nverts; ++t) {
                const double a = v0[3 * (uint64_t)verts[t] + c];
                const double b = v1[3 * (uint64_t)verts[t] + c];
                /* std::min/max semantics: min(lo, a) = (a < lo) ? a : lo */
                lo = (a < lo) ? a : lo;
                hi = (hi < a) ? a : hi;
                lo = (b < lo) ? b : lo;
                hi = (hi < b) ? b : hi;
            }
            if (inflation > 0.0) {
                double pad = inflation * (hi - lo);
                if (pad == 0.0)
                    pad = 1e-12;
                lo -= pad;
                hi += pad;
            }
            if (!isfinite(lo) || !isfinite(hi))
                return CCDK_INVALID_INPUT; /* round_*_reduced throw, aabb.cpp:12-13 */
            mn[3 * s + c] = orc_round_down_reduced(lo);
            mx[3 * s + c] = orc_round_up_reduced(hi);
        }
    }
    return 0;
}

/* ------------------------------------------------------------- broad phase */

/* choose_axis, broadphase.cpp:45-67: serial mean, serial variance, strict >. */
int orc_choose_axis(const float* mn, const float* mx, uint64_t k)
{
    double mean[3] = { 0, 0, 0 }, var[3] = { 0, 0, 0 };
    for (uint64_t i = 0; i < k; ++i)
        for (int c = 0; c < 3; ++c)
            mean[c] += ((double)mn[3 * i + c] + mx[3 * i + c]) / 2.0;
    for (int c = 0; c < 3; ++c)
        mean[c] /= (double)k;
    for (uint64_t i = 0; i < k; ++i)
        for (int c = 0; c < 3; ++c) {
            const double d = ((double)mn[3 * i + c] + mx[3 * i + c]) / 2.0 - mean[c];
            var[c] += d * d;
        }
    int axis = 0;
    for (int c = 1; c < 3; ++c)
        if (var[c] > var[axis])
            axis = c;
    return axis;
}

typedef struct {
    const float* mn;
    const uint8_t* kind;
    const uint32_t* index;
    int axis;
} sort_ctx;

static sort_ctx g_sort; /* qsort has no context argument in C11 */

/* sort_positions comparator, broadphase.cpp:23-35: min on axis, float !=,
 * then owner (kind, index). */
static int cmp_positions(const void* pa, const void* pb)
{
    const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    const float ma = g_sort.mn[3 * (uint64_t)a + g_sort.axis];
    const float mb = g_sort.mn[3 * (uint64_t)b + g_sort.axis];
    if (ma != mb)
        return ma < mb ? -1 : 1;
    const uint64_t oa = ((uint64_t)g_sort.kind[a] << 32) | g_sort.index[a];
    const uint64_t ob = ((uint64_t)g_sort.kind[b] << 32) | g_sort.index[b];
    return oa < ob ? -1 : (oa > ob ? 1 : 0);
}

static int cmp_pair(const void* pa, const void* pb)
{
    const uint64_t* a = (const uint64_t*)pa;
    const uint64_t* b = (const uint64_t*)pb;
    if (a[0] != b[0])
        return a[0] < b[0] ? -1 : 1;
    return a[1] < b[1] ? -1 : (a[1] > b[1] ? 1 : 0);
}

static int prim_vertices(uint8_t kind, uint32_t index, const uint32_t* e, const uint32_t* f,
                         uint32_t out[3])
{
    if (kind == CCDK_KIND_VERTEX) {
        out[0] = index;
        return 1;
    }
    if (kind == CCDK_KIND_EDGE) {
        out[0] = e[2 * (uint64_t)index];
        out[1] = e[2 * (uint64_t)index + 1];
        return 2;
    }
    out[0] = f[3 * (uint64_t)index];
    out[1] = f[3 * (uint64_t)index + 1];
    out[2] = f[3 * (uint64_t)index + 2];
    return 3;
}

/* keep_pair, broadphase.cpp:12-20, with share_vertex, scene.cpp:53-78. */
static int keep_pair(uint8_t ka, uint32_t ia, uint8_t kb, uint32_t ib, const uint32_t* e,
                     const uint32_t* f)
{
    const int vf = (ka == CCDK_KIND_VERTEX && kb == CCDK_KIND_FACE)
        || (ka == CCDK_KIND_FACE && kb == CCDK_KIND_VERTEX);
    const int ee = ka == CCDK_KIND_EDGE && kb == CCDK_KIND_EDGE;
    if (!vf && !ee)
        return 0;
    uint32_t va[3], vb[3];
    const int na = prim_vertices(ka, ia, e, f, va);
    const int nb = prim_vertices(kb, ib, e, f, vb);
    for (int i = 0; i < na; ++i)
        for (int j = 0; j < nb; ++j)
            if (va[i] == vb[j])
                return 0;
    return 1;
}

typedef struct {
    uint64_t* data;
    uint64_t n, cap;
} u64vec;

static void push2(u64vec* v, uint64_t a, uint64_t b)
{
    if (v->n + 2 > v->cap) {
        v->cap = v->cap ? 2 * v->cap : 1024;
        v->data = (uint64_t*)realloc(v->data, v->cap * sizeof(uint64_t));
    }
    v->data[v->n++] = a;
    v->data[v->n++] = b;
}

/* make_pair_canonical (broadphase.hpp:21-24) + finalize (broadphase.cpp:37-41). */
static void emit(u64vec* out, uint8_t ka, uint32_t ia, uint8_t kb, uint32_t ib)
{
    const uint64_t a = ((uint64_t)ka << 32) | ia;
    const uint64_t b = ((uint64_t)kb << 32) | ib;
    if (a < b)
        push2(out, a, b);
    else
        push2(out, b, a);
}

static void finalize_pairs(u64vec* v)
{
    const uint64_t np = v->n / 2;
    if (np == 0)
        return;
    qsort(v->data, np, 2 * sizeof(uint64_t), cmp_pair);
    uint64_t w = 1;
    for (uint64_t i = 1; i < np; ++i)
        if (v->data[2 * i] != v->data[2 * (w - 1)] || v->data[2 * i + 1] != v->data[2 * (w - 1) + 1]) {
            v->data[2 * w] = v->data[2 * i];
            v->data[2 * w + 1] = v->data[2 * i + 1];
            ++w;
        }
    v->n = 2 * w;
}

static int overlaps_axis(const float* mn, const float* mx, uint64_t a, uint64_t b, int c)
{
    /* Aabb::overlaps_axis, aabb.hpp:34-38 */
    return mn[3 * a + c] <= mx[3 * b + c] && mn[3 * b + c] <= mx[3 * a + c];
}

/* stq (broadphase.cpp:69-127) and sap (156-192) produce the same set: for
 * each sorted left position i in the range, every later j with
 * min_axis[j] <= max_axis[i], kept when ax1/ax2 overlap and keep_pair holds.
 * StqStats: the queue entry (i, j) lives in round j-i-1, so
 * round_sizes[r] = #{i : run_len(i) >= r+1}.
 * bf (129-154) ranges over raw positions and tests all three axes. */
int orc_broad(int method, const float* mn, const float* mx, const uint8_t* kind,
              const uint32_t* index, uint64_t k, const uint32_t* e, uint64_t ne,
              const uint32_t* f, uint64_t nf, uint64_t rb, uint64_t re, uint64_t** pairs,
              uint64_t* npairs, uint64_t** rounds, uint64_t* nrounds, uint64_t* max_queue)
{
    (void)ne;
    (void)nf;
    u64vec out = { 0, 0, 0 };
    if (rounds)
        *rounds = NULL;
    if (nrounds)
        *nrounds = 0;
    if (max_queue)
        *max_queue = 0;
    if (method == CCDK_BROAD_BF) {
        const uint64_t b = rb < k ? rb : k, en = re < k ? re : k;
        for (uint64_t i = b; i < en; ++i)
            for (uint64_t j = i + 1; j < k; ++j)
                if (overlaps_axis(mn, mx, i, j, 0) && overlaps_axis(mn, mx, i, j, 1)
                    && overlaps_axis(mn, mx, i, j, 2)
                    && keep_pair(kind[i], index[i], kind[j], index[j], e, f))
                    emit(&out, kind[i], index[i], kind[j], index[j]);
    } else if (k >= 2) {
        const int axis = orc_choose_axis(mn, mx, k);
        const int ax1 = (axis + 1) % 3, ax2 = (axis + 2) % 3;
        uint32_t* order = (uint32_t*)malloc(k * sizeof(uint32_t));
        for (uint64_t i = 0; i < k; ++i)
            order[i] = (uint32_t)i;
        g_sort.mn = mn;
        g_sort.kind = kind;
        g_sort.index = index;
        g_sort.axis = axis;
        qsort(order, k, sizeof(uint32_t), cmp_positions);
        /* STQ seeds left positions [min(b,k-1), min(e,k-1)) (broadphase.cpp:85-90);
         * SAP uses [min(b,k), min(e,k)); position k-1 has no partner either way. */
        const uint64_t lo = rb < k - 1 ? rb : k - 1;
        const uint64_t hi = re < k - 1 ? re : k - 1;
        uint64_t* hist = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
        uint64_t max_run = 0;
        for (uint64_t i = lo; i < hi; ++i) {
            const uint64_t a = order[i];
            const float reach = mx[3 * a + axis];
            uint64_t j = i + 1;
            for (; j < k; ++j) {
                const uint64_t b = order[j];
                if (mn[3 * b + axis] > reach)
                    break;
                if (overlaps_axis(mn, mx, a, b, ax1) && overlaps_axis(mn, mx, a, b, ax2)
                    && keep_pair(kind[a], index[a], kind[b], index[b], e, f))
                    emit(&out, kind[a], index[a], kind[b], index[b]);
            }
            const uint64_t run = j - i - 1;
            hist[run] += 1;
            if (run > max_run)
                max_run = run;
        }
        if (rounds && method == CCDK_BROAD_STQ) {
            uint64_t* r = (uint64_t*)malloc((max_run ? max_run : 1) * sizeof(uint64_t));
            uint64_t acc = 0;
            for (uint64_t x = max_run; x >= 1; --x) {
                acc += hist[x];
                r[x - 1] = acc;
            }
            *rounds = r;
            *nrounds = max_run;
            *max_queue = max_run ? r[0] : 0;
        }
        free(hist);
        free(order);
    }
    finalize_pairs(&out);
    *npairs = out.n / 2;
    *pairs = out.data ? out.data : (uint64_t*)malloc(16);
    return 0;
}

/* classify, broadphase.cpp:194-239: range check, VF and EE gathers, other
 * kinds dropped; output VF block then EE block (pipeline.cpp:162-165). */
int orc_classify(const uint64_t* pairs, uint64_t np, const double* v0, const double* v1,
                 uint64_t nv, const uint32_t* e, uint64_t ne, const uint32_t* f,
                 uint64_t nf, uint8_t* kind_out, double* points_out, uint64_t* source_out,
                 uint64_t* n_vf, uint64_t* n_ee)
{
    uint64_t w = 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (uint64_t i = 0; i < np; ++i) {
            const uint64_t ids[2] = { pairs[2 * i], pairs[2 * i + 1] };
            for (int s = 0; s < 2; ++s) {
                const uint32_t kd = (uint32_t)(ids[s] >> 32), ix = (uint32_t)ids[s];
                const uint64_t limit = kd == 0 ? nv : kd == 1 ? ne : nf;
                if (ix >= limit)
                    return CCDK_INVALID_INPUT;
            }
            const uint8_t ka = (uint8_t)(ids[0] >> 32), kb = (uint8_t)(ids[1] >> 32);
            const uint32_t ia = (uint32_t)ids[0], ib = (uint32_t)ids[1];
            uint32_t pv[4];
            if (pass == 0 && ka == CCDK_KIND_VERTEX && kb == CCDK_KIND_FACE) {
                if (!keep_pair(ka, ia, kb, ib, e, f))
                    continue;
                pv[0] = ia;
                pv[1] = f[3 * (uint64_t)ib];
                pv[2] = f[3 * (uint64_t)ib + 1];
                pv[3] = f[3 * (uint64_t)ib + 2];
                kind_out[w] = CCDK_QUERY_VF;
            } else if (pass == 1 && ka == CCDK_KIND_EDGE && kb == CCDK_KIND_EDGE) {
                if (!keep_pair(ka, ia, kb, ib, e, f))
                    continue;
                pv[0] = e[2 * (uint64_t)ia];
                pv[1] = e[2 * (uint64_t)ia + 1];
                pv[2] = e[2 * (uint64_t)ib];
                pv[3] = e[2 * (uint64_t)ib + 1];
                kind_out[w] = CCDK_QUERY_EE;
            } else {
                continue;
            }
            for (int p = 0; p < 4; ++p)
                for (int c = 0; c < 3; ++c) {
                    points_out[24 * w + 3 * p + c] = v0[3 * (uint64_t)pv[p] + c];
                    points_out[24 * w + 12 + 3 * p + c] = v1[3 * (uint64_t)pv[p] + c];
                }
            source_out[2 * w] = ids[0];
            source_out[2 * w + 1] = ids[1];
            ++w;
        }
        if (pass == 0)
            *n_vf = w;
    }
    *n_ee = w - *n_vf;
    return 0;
}

/* ------------------------------------------------------ interval arithmetic */

/* interval.hpp:16-92.  Outward widening by one representable step
 * (nextafter toward +/-inf), with |x| < 1e-250 flushed to +/-1e-250 and NaN
 * left as is (interval.hpp:34-49). */
#define KFLUSH 1e-250

static double wup(double x)
{
    if (isnan(x))
        return x;
    if (x < KFLUSH && x > -KFLUSH)
        return KFLUSH;
    return nextafter(x, INFINITY);
}

static double wdown(double x) { return -wup(-x); }

typedef struct {
    double lo, hi;
} ival;

static ival iv_point(double x)
{
    ival r = { x, x };
    return r;
}

static ival iv_add(ival a, ival b)
{
    ival r = { wdown(a.lo + b.lo), wup(a.hi + b.hi) };
    return r;
}

static ival iv_sub(ival a, ival b)
{
    ival r = { wdown(a.lo - b.hi), wup(a.hi - b.lo) };
    return r;
}

/* scale_nn, narrowphase.cpp:30-33: exact non-negative point factor. */
static ival iv_scale(double p, ival a)
{
    ival r = { wdown(p * a.lo), wup(p * a.hi) };
    return r;
}

static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* ---------------------------------------------------------- narrow phase */

typedef struct {
    double tlo, thi, ulo, uhi, vlo, vhi;
    uint16_t depth[3];
    uint32_t q;
} obox;

typedef struct {
    ival corner[8][3]; /* bit0 = t, bit1 = u, bit2 = v */
    ival range[3];
} oeval;

/* evaluate_box, narrowphase.cpp:35-85, in the reference's literal form. */
static void evaluate(uint8_t kind, const double* P, const obox* b, oeval* ev)
{
    const double* x0 = P;      /* points_t0[p][c] = x0[3p+c] */
    const double* x1 = P + 12; /* points_t1 */
    ival delta[4][3];
    for (int p = 0; p < 4; ++p)
        for (int c = 0; c < 3; ++c)
            delta[p][c] = iv_sub(iv_point(x1[3 * p + c]), iv_point(x0[3 * p + c]));
    const int vf = kind == CCDK_QUERY_VF;
    const int origin = vf ? 1 : 2, u_from = vf ? 1 : 0, u_to = vf ? 2 : 1;
    ival base[2][3], du[2][3], dv[2][3];
    for (int tb = 0; tb < 2; ++tb) {
        const double t = tb ? b->thi : b->tlo;
        ival at[4][3];
        for (int p = 0; p < 4; ++p)
            for (int c = 0; c < 3; ++c)
                at[p][c] = iv_add(iv_point(x0[3 * p + c]), iv_scale(t, delta[p][c]));
        for (int c = 0; c < 3; ++c) {
            base[tb][c] = iv_sub(at[0][c], at[origin][c]);
            du[tb][c] = iv_sub(at[u_to][c], at[u_from][c]);
            dv[tb][c] = iv_sub(at[3][c], at[origin][c]);
        }
    }
    for (int corner = 0; corner < 8; ++corner) {
        const int tb = corner & 1;
        const double u = (corner & 2) ? b->uhi : b->ulo;
        const double v = (corner & 4) ? b->vhi : b->vlo;
        for (int c = 0; c < 3; ++c) {
            const ival ut = iv_scale(u, du[tb][c]);
            const ival s = vf ? iv_sub(base[tb][c], ut) : iv_add(base[tb][c], ut);
            ev->corner[corner][c] = iv_sub(s, iv_scale(v, dv[tb][c]));
        }
        for (int c = 0; c < 3; ++c) {
            if (corner == 0) {
                ev->range[c] = ev->corner[0][c];
            } else {
                ev->range[c].lo = dmin(ev->range[c].lo, ev->corner[corner][c].lo);
                ev->range[c].hi = dmax(ev->range[c].hi, ev->corner[corner][c].hi);
            }
        }
    }
}

void orc_inclusion_box(uint8_t kind, const double* points, const double* box, double* out)
{
    obox b = { box[0], box[1], box[2], box[3], box[4], box[5], { 0, 0, 0 }, 0 };
    oeval ev;
    evaluate(kind, points, &b, &ev);
    for (int c = 0; c < 3; ++c) {
        out[2 * c] = ev.range[c].lo;
        out[2 * c + 1] = ev.range[c].hi;
    }
}

static int splittable(double lo, double hi)
{
    /* narrowphase.cpp:109-113 */
    const double mid = lo + 0.5 * (hi - lo);
    return mid > lo && mid < hi;
}

static double* dim_lo(obox* b, int d) { return d == 0 ? &b->tlo : d == 1 ? &b->ulo : &b->vlo; }
static double* dim_hi(obox* b, int d) { return d == 0 ? &b->thi : d == 1 ? &b->uhi : &b->vhi; }

/* process_interval, narrowphase.cpp:134-187 (influences 89-107, split_box
 * 122-132).  action: 0 pruned, 1 collision, 2 split. */
static int process(uint8_t kind, const double* P, const obox* b, double t_star, double d,
                   const ccdk_narrow_cfg* cfg, double* cand_t, int* zdiag, obox* kids,
                   int* evaluated)
{
    *zdiag = 0;
    *evaluated = 0;
    if (b->tlo >= t_star || b->tlo >= cfg->t_max)
        return 0;
    if (kind == CCDK_QUERY_VF && b->ulo + b->vlo > 1.0)
        return 0;
    oeval ev;
    evaluate(kind, P, b, &ev);
    *evaluated = 1;
    for (int c = 0; c < 3; ++c)
        if (ev.range[c].lo > d || ev.range[c].hi < -d)
            return 0;
    const int force_zero = cfg->no_zero_toi && b->tlo == 0.0;
    if (!force_zero) {
        int inside = 1;
        double wmax = ev.range[0].hi - ev.range[0].lo;
        for (int c = 0; c < 3; ++c) {
            inside = inside && ev.range[c].lo >= -d && ev.range[c].hi <= d;
            wmax = dmax(wmax, ev.range[c].hi - ev.range[c].lo);
        }
        if (wmax < cfg->delta || inside) {
            *cand_t = b->tlo;
            return 1;
        }
    }
    double infl[3] = { 0, 0, 0 };
    for (int dd = 0; dd < 3; ++dd) {
        const int bit = 1 << dd;
        for (int corner = 0; corner < 8; ++corner) {
            if (corner & bit)
                continue;
            for (int c = 0; c < 3; ++c) {
                const ival a = ev.corner[corner][c], bb = ev.corner[corner | bit][c];
                const double diff = fabs(0.5 * (bb.lo + bb.hi) - 0.5 * (a.lo + a.hi));
                infl[dd] = dmax(infl[dd], diff);
            }
        }
    }
    obox tmp = *b;
    int dim = -1;
    for (int dd = 0; dd < 3; ++dd) {
        if (!splittable(*dim_lo(&tmp, dd), *dim_hi(&tmp, dd)))
            continue;
        if (dim < 0 || infl[dd] > infl[dim])
            dim = dd;
    }
    if (dim < 0) {
        *cand_t = b->tlo;
        *zdiag = force_zero;
        return 1;
    }
    const double lo = *dim_lo(&tmp, dim), hi = *dim_hi(&tmp, dim);
    const double mid = lo + 0.5 * (hi - lo);
    kids[0] = *b;
    kids[1] = *b;
    *dim_hi(&kids[0], dim) = mid;
    *dim_lo(&kids[1], dim) = mid;
    kids[0].depth[dim]++;
    kids[1].depth[dim]++;
    return 2;
}

void orc_process_interval(uint8_t kind, const double* points, const double* box,
                          const uint16_t* depth, double t_star, double sep,
                          const ccdk_narrow_cfg* cfg, uint8_t* action, double* cand_t,
                          uint8_t* zdiag, double* children, uint16_t* child_depth)
{
    obox b = { box[0], box[1], box[2], box[3], box[4], box[5],
               { depth[0], depth[1], depth[2] }, 0 };
    obox kids[2];
    memset(kids, 0, sizeof kids);
    kids[0].thi = kids[0].uhi = kids[0].vhi = 1.0;
    kids[1] = kids[0];
    double ct = INFINITY;
    int zd = 0, evald = 0;
    const double d = sep >= 0.0 ? sep : cfg->min_separation;
    const int a = process(kind, points, &b, t_star, d, cfg, &ct, &zd, kids, &evald);
    *action = (uint8_t)a;
    *cand_t = ct;
    *zdiag = (uint8_t)zd;
    for (int ch = 0; ch < 2; ++ch) {
        const double v[6] = { kids[ch].tlo, kids[ch].thi, kids[ch].ulo,
                              kids[ch].uhi, kids[ch].vlo, kids[ch].vhi };
        memcpy(children + 6 * ch, v, sizeof v);
        for (int dd = 0; dd < 3; ++dd)
            child_depth[3 * ch + dd] = kids[ch].depth[dd];
    }
}

typedef struct {
    obox* data;
    uint64_t n, cap;
} boxvec;

static void bpush(boxvec* v, const obox* b)
{
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 1024;
        v->data = (obox*)realloc(v->data, v->cap * sizeof(obox));
    }
    v->data[v->n++] = *b;
}

/* NarrowConfig::validate, narrowphase.cpp:10-20. */
static int validate_ncfg(const ccdk_narrow_cfg* c)
{
    if (!(c->delta > 0.0) || c->max_splits < 1 || c->min_separation < 0.0
        || !(c->t_max > 0.0) || c->t_max > 1.0)
        return CCDK_CONFIG;
    return 0;
}

/* narrow_phase, narrowphase.cpp:189-311: one root box per query, whole
 * generations processed against a per-query ToI snapshot taken at the
 * generation start, then a serial fold in queue order with the per-query
 * split budget and exhaustion compaction. */
int orc_narrow_phase(const uint8_t* kind, const double* points, uint64_t n,
                     const double* seps, const ccdk_narrow_cfg* cfg, uint64_t capacity,
                     double* toi, uint8_t* flags, ccdk_narrow_stats* st)
{
    if (validate_ncfg(cfg))
        return CCDK_CONFIG;
    memset(st, 0, sizeof *st);
    st->global_toi = INFINITY;
    for (uint64_t q = 0; q < n; ++q) {
        toi[q] = INFINITY;
        flags[q] = 0;
    }
    if (n == 0)
        return 0;
    if (n > capacity) {
        st->overflow = 1;
        return 0;
    }
    boxvec cur = { 0, 0, 0 }, nxt = { 0, 0, 0 };
    for (uint64_t q = 0; q < n; ++q) {
        obox r = { 0, 1, 0, 1, 0, 1, { 0, 0, 0 }, (uint32_t)q };
        bpush(&cur, &r);
    }
    uint64_t* used = (uint64_t*)calloc(n, sizeof(uint64_t));
    uint8_t* done = (uint8_t*)calloc(n, 1);
    double* snap = (double*)malloc(n * sizeof(double));
    int ret = 0;
    while (cur.n) {
        if (cur.n > st->peak_queue)
            st->peak_queue = cur.n;
        memcpy(snap, toi, n * sizeof(double));
        st->generations++;
        nxt.n = 0;
        int any_exhausted = 0;
        for (uint64_t i = 0; i < cur.n; ++i) {
            const obox* b = &cur.data[i];
            const uint32_t q = b->q;
            if (done[q])
                continue;
            const double d = seps ? seps[q] : cfg->min_separation;
            double ct = INFINITY;
            int zd = 0, evald = 0;
            obox kids[2];
            const int a = process(kind[q], points + 24 * (uint64_t)q, b, snap[q], d, cfg, &ct,
                                  &zd, kids, &evald);
            st->evaluations += (uint64_t)evald;
            if (a == 1) {
                toi[q] = dmin(toi[q], ct);
                if (zd)
                    flags[q] |= CCDK_FLAG_ZERO_TOI_DIAG;
            } else if (a == 2) {
                st->split_actions++;
                const int exempt = cfg->no_zero_toi && b->tlo == 0.0;
                if (exempt || used[q] < cfg->max_splits) {
                    if (!exempt) {
                        used[q]++;
                        st->total_splits++;
                    }
                    kids[0].q = kids[1].q = q;
                    bpush(&nxt, &kids[0]);
                    bpush(&nxt, &kids[1]);
                } else {
                    toi[q] = dmin(toi[q], b->tlo);
                    flags[q] |= CCDK_FLAG_TOLERANCE_HIT;
                    if (cfg->no_zero_toi && b->tlo == 0.0)
                        flags[q] |= CCDK_FLAG_ZERO_TOI_DIAG;
                    any_exhausted = 1;
                }
            }
        }
        if (any_exhausted) {
            uint64_t w = 0;
            for (uint64_t i = 0; i < nxt.n; ++i) {
                const uint32_t q = nxt.data[i].q;
                if (flags[q] & CCDK_FLAG_TOLERANCE_HIT) {
                    toi[q] = dmin(toi[q], nxt.data[i].tlo);
                    if (cfg->no_zero_toi && nxt.data[i].tlo == 0.0)
                        flags[q] |= CCDK_FLAG_ZERO_TOI_DIAG;
                } else {
                    nxt.data[w++] = nxt.data[i];
                }
            }
            nxt.n = w;
            for (uint64_t q = 0; q < n; ++q)
                if (flags[q] & CCDK_FLAG_TOLERANCE_HIT)
                    done[q] = 1;
        }
        if (nxt.n > capacity) {
            st->overflow = 1;
            for (uint64_t q = 0; q < n; ++q) {
                toi[q] = INFINITY;
                flags[q] = 0;
            }
            ret = 0;
            goto out;
        }
        if (nxt.n > st->peak_queue)
            st->peak_queue = nxt.n;
        boxvec t = cur;
        cur = nxt;
        nxt = t;
    }
    for (uint64_t q = 0; q < n; ++q)
        st->global_toi = dmin(st->global_toi, toi[q]);
out:
    free(cur.data);
    free(nxt.data);
    free(used);
    free(done);
    free(snap);
    return ret;
}

/* ccd (pipeline.cpp:218-232) through run_batched (179-216) at the default,
 * effectively unbounded budget, Absolute min-separation (39-55). */
int orc_ccd(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
            uint64_t ne, const uint32_t* f, uint64_t nf, const ccdk_pipeline_cfg* cfg,
            ccdk_report* rep, uint64_t** pairs_out)
{
    if (validate_ncfg(&cfg->narrow) || cfg->inflation < 0.0 || cfg->threads < 1
        || cfg->memory_budget <= cfg->rs_params)
        return CCDK_CONFIG;
    if (validate_scene(v0, v1, nv, e, ne, f, nf))
        return CCDK_INVALID_INPUT;
    memset(rep, 0, sizeof *rep);
    rep->toi = INFINITY;
    const uint64_t k = nv + ne + nf;
    float* mn = (float*)malloc((k ? k : 1) * 3 * sizeof(float));
    float* mx = (float*)malloc((k ? k : 1) * 3 * sizeof(float));
    uint8_t* kind = (uint8_t*)malloc(k ? k : 1);
    uint32_t* index = (uint32_t*)malloc((k ? k : 1) * sizeof(uint32_t));
    int rc = orc_build_boxes(v0, v1, nv, e, ne, f, nf, cfg->inflation, mn, mx, kind, index);
    uint64_t* pairs = NULL;
    uint64_t np = 0;
    if (!rc)
        rc = orc_broad(cfg->broad_method, mn, mx, kind, index, k, e, ne, f, nf, 0, UINT64_MAX,
                       &pairs, &np, NULL, NULL, NULL);
    if (!rc) {
        uint8_t* qk = (uint8_t*)malloc(np ? np : 1);
        double* qp = (double*)malloc((np ? np : 1) * 24 * sizeof(double));
        uint64_t* src = (uint64_t*)malloc((np ? np : 1) * 2 * sizeof(uint64_t));
        uint64_t nvf = 0, nee = 0;
        rc = orc_classify(pairs, np, v0, v1, nv, e, ne, f, nf, qk, qp, src, &nvf, &nee);
        const uint64_t nq = nvf + nee;
        if (!rc && nq) {
            double* toi = (double*)malloc(nq * sizeof(double));
            uint8_t* fl = (uint8_t*)malloc(nq);
            ccdk_narrow_stats st;
            rc = orc_narrow_phase(qk, qp, nq, NULL, &cfg->narrow, UINT64_MAX, toi, fl, &st);
            for (uint64_t q = 0; q < nq && !rc; ++q) {
                rep->toi = dmin(rep->toi, toi[q]);
                rep->tolerance_hit |= (fl[q] & CCDK_FLAG_TOLERANCE_HIT) != 0;
                rep->zero_toi_diagnostic |= (fl[q] & CCDK_FLAG_ZERO_TOI_DIAG) != 0;
            }
            rep->total_splits = st.total_splits;
            rep->peak_queue = st.peak_queue;
            rep->evaluations = st.evaluations;
            rep->split_actions = st.split_actions;
            rep->generations = st.generations;
            free(toi);
            free(fl);
        }
        rep->candidate_count = np;
        rep->query_count = nq;
        rep->vf_count = nvf;
        rep->batch_count = 1;
        free(qk);
        free(qp);
        free(src);
    }
    if (pairs_out)
        *pairs_out = pairs;
    else
        free(pairs);
    free(mn);
    free(mx);
    free(kind);
    free(index);
    return rc;
}
