// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" adapter over the UNMODIFIED reference ccdkit sources, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/
// libccdref.so with -Dccdkit=ccdkit_ref (the namespace rename lets the
// reference and the product link side by side).  Only tests/,
// __graft_entry__.smoke() and bench.py's reference/cpu_baseline arm load it.
//
// Array layouts follow include/ccdk.h.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ccdkit/aabb.hpp"
#include "ccdkit/bench.hpp"
#include "ccdkit/broadphase.hpp"
#include "ccdkit/distance.hpp"
#include "ccdkit/narrowphase.hpp"
#include "ccdkit/pipeline.hpp"
#include "ccdkit/scene.hpp"

#include "ccdk.h"

using namespace ccdkit_ref;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what)
{
    g_err = what;
    return code;
}

template <typename F>
int guard(F&& f)
{
    try {
        f();
        return 0;
    } catch (const InvalidInput& e) {
        return fail(CCDK_INVALID_INPUT, e.what());
    } catch (const ConfigError& e) {
        return fail(CCDK_CONFIG, e.what());
    } catch (const std::exception& e) {
        return fail(99, e.what());
    }
}

SceneStep make_scene(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                     uint64_t ne, const uint32_t* f, uint64_t nf)
{
    SceneStep s;
    s.vertices_t0.resize(nv);
    s.vertices_t1.resize(nv);
    for (uint64_t i = 0; i < nv; ++i)
        for (int c = 0; c < 3; ++c) {
            s.vertices_t0[i][c] = v0[3 * i + c];
            s.vertices_t1[i][c] = v1[3 * i + c];
        }
    s.edges.resize(ne);
    for (uint64_t i = 0; i < ne; ++i)
        s.edges[i] = { e[2 * i], e[2 * i + 1] };
    s.faces.resize(nf);
    for (uint64_t i = 0; i < nf; ++i)
        s.faces[i] = { f[3 * i], f[3 * i + 1], f[3 * i + 2] };
    return s;
}

std::vector<Aabb> make_boxes(const float* mn, const float* mx, const uint8_t* kind,
                             const uint32_t* index, uint64_t k)
{
    std::vector<Aabb> boxes(k);
    for (uint64_t i = 0; i < k; ++i) {
        for (int c = 0; c < 3; ++c) {
            boxes[i].min_corner[c] = mn[3 * i + c];
            boxes[i].max_corner[c] = mx[3 * i + c];
        }
        boxes[i].owner = { static_cast<PrimitiveKind>(kind[i]), index[i] };
    }
    return boxes;
}

uint64_t pack_id(PrimitiveId id)
{
    return (static_cast<uint64_t>(id.kind) << 32) | id.index;
}

PrimitiveId unpack_id(uint64_t v)
{
    return { static_cast<PrimitiveKind>(v >> 32), static_cast<uint32_t>(v) };
}

NarrowQuery make_query(uint8_t kind, const double* p)
{
    NarrowQuery q;
    q.kind = kind ? QueryKind::EdgeEdge : QueryKind::VertexFace;
    for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) {
            q.points_t0[i][c] = p[3 * i + c];
            q.points_t1[i][c] = p[12 + 3 * i + c];
        }
    return q;
}

void store_query(const NarrowQuery& q, uint8_t* kind, double* p)
{
    *kind = q.kind == QueryKind::EdgeEdge ? 1 : 0;
    for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) {
            p[3 * i + c] = q.points_t0[i][c];
            p[12 + 3 * i + c] = q.points_t1[i][c];
        }
}

NarrowConfig make_ncfg(const ccdk_narrow_cfg* c)
{
    NarrowConfig n;
    n.delta = c->delta;
    n.min_separation = c->min_separation;
    n.t_max = c->t_max;
    n.max_splits = c->max_splits;
    n.no_zero_toi = c->no_zero_toi != 0;
    return n;
}

PipelineConfig make_pcfg(const ccdk_pipeline_cfg* c)
{
    PipelineConfig p;
    p.narrow = make_ncfg(&c->narrow);
    p.broad_method = static_cast<BroadMethod>(c->broad_method);
    p.memory_budget = c->memory_budget;
    p.record_sizes.params = c->rs_params;
    p.record_sizes.query = c->rs_query;
    p.record_sizes.interval = c->rs_interval;
    p.record_sizes.pair_ints = c->rs_pair_ints;
    p.min_sep_mode = static_cast<MinSepMode>(c->min_sep_mode);
    p.min_sep_fraction = c->min_sep_fraction;
    p.threads = c->threads;
    p.inflation = c->inflation;
    return p;
}

template <typename T>
T* dup(const std::vector<T>& v)
{
    T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size() * sizeof(T))));
    if (!v.empty())
        std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

void scene_out(const SceneStep& s, double** v0, double** v1, uint64_t* nv, uint32_t** e,
               uint64_t* ne, uint32_t** f, uint64_t* nf)
{
    std::vector<double> a, b;
    for (size_t i = 0; i < s.vertices_t0.size(); ++i)
        for (int c = 0; c < 3; ++c) {
            a.push_back(s.vertices_t0[i][c]);
            b.push_back(s.vertices_t1[i][c]);
        }
    std::vector<uint32_t> ev, fv;
    for (const auto& x : s.edges) {
        ev.push_back(x[0]);
        ev.push_back(x[1]);
    }
    for (const auto& x : s.faces) {
        fv.push_back(x[0]);
        fv.push_back(x[1]);
        fv.push_back(x[2]);
    }
    *v0 = dup(a);
    *v1 = dup(b);
    *e = dup(ev);
    *f = dup(fv);
    *nv = s.vertices_t0.size();
    *ne = s.edges.size();
    *nf = s.faces.size();
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_round(const double* x, uint64_t n, float* down, float* up)
{
    return guard([&] {
        for (uint64_t i = 0; i < n; ++i) {
            down[i] = round_down_reduced(x[i]);
            up[i] = round_up_reduced(x[i]);
        }
    });
}

int ref_build_boxes(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                    uint64_t ne, const uint32_t* f, uint64_t nf, double inflation,
                    unsigned threads, float* mn, float* mx, uint8_t* kind, uint32_t* index)
{
    return guard([&] {
        const SceneStep s = make_scene(v0, v1, nv, e, ne, f, nf);
        const std::vector<Aabb> boxes = build_boxes(s, inflation, threads);
        for (size_t i = 0; i < boxes.size(); ++i) {
            for (int c = 0; c < 3; ++c) {
                mn[3 * i + c] = boxes[i].min_corner[c];
                mx[3 * i + c] = boxes[i].max_corner[c];
            }
            kind[i] = static_cast<uint8_t>(boxes[i].owner.kind);
            index[i] = boxes[i].owner.index;
        }
    });
}

int ref_choose_axis(const float* mn, const float* mx, uint64_t k, int* axis)
{
    return guard([&] {
        std::vector<uint8_t> kind(k, 0);
        std::vector<uint32_t> idx(k, 0);
        *axis = choose_axis(make_boxes(mn, mx, kind.data(), idx.data(), k));
    });
}

int ref_broad(int method, const float* mn, const float* mx, const uint8_t* kind,
              const uint32_t* index, uint64_t k, const double* v0, const double* v1,
              uint64_t nv, const uint32_t* e, uint64_t ne, const uint32_t* f, uint64_t nf,
              unsigned threads, uint64_t rb, uint64_t re, uint64_t** pairs,
              uint64_t* npairs, uint64_t** rounds, uint64_t* nrounds, uint64_t* max_queue)
{
    return guard([&] {
        const SceneStep s = make_scene(v0, v1, nv, e, ne, f, nf);
        const std::vector<Aabb> boxes = make_boxes(mn, mx, kind, index, k);
        const SweepRange range { static_cast<size_t>(rb), static_cast<size_t>(re) };
        std::vector<CandidatePair> out;
        StqStats stats;
        if (method == CCDK_BROAD_STQ)
            out = stq(boxes, s, threads, &stats, range);
        else if (method == CCDK_BROAD_BF)
            out = bf(boxes, s, threads, range);
        else
            out = sap(boxes, s, threads, range);
        std::vector<uint64_t> flat;
        flat.reserve(out.size() * 2);
        for (const auto& p : out) {
            flat.push_back(pack_id(p.left));
            flat.push_back(pack_id(p.right));
        }
        *pairs = dup(flat);
        *npairs = out.size();
        std::vector<uint64_t> r(stats.round_sizes.begin(), stats.round_sizes.end());
        if (rounds)
            *rounds = dup(r);
        if (nrounds)
            *nrounds = r.size();
        if (max_queue)
            *max_queue = stats.max_queue;
    });
}

int ref_classify(const uint64_t* pairs, uint64_t np, const double* v0, const double* v1,
                 uint64_t nv, const uint32_t* e, uint64_t ne, const uint32_t* f,
                 uint64_t nf, uint8_t* kind_out, double* points_out, uint64_t* source_out,
                 uint64_t* n_vf, uint64_t* n_ee)
{
    return guard([&] {
        const SceneStep s = make_scene(v0, v1, nv, e, ne, f, nf);
        std::vector<CandidatePair> cp(np);
        for (uint64_t i = 0; i < np; ++i)
            cp[i] = { unpack_id(pairs[2 * i]), unpack_id(pairs[2 * i + 1]) };
        const ClassifiedQueries cq = classify(cp, s);
        uint64_t w = 0;
        for (const auto* list : { &cq.vertex_face, &cq.edge_edge })
            for (const NarrowQuery& q : *list) {
                store_query(q, &kind_out[w], &points_out[24 * w]);
                source_out[2 * w] = pack_id(q.source.left);
                source_out[2 * w + 1] = pack_id(q.source.right);
                ++w;
            }
        *n_vf = cq.vertex_face.size();
        *n_ee = cq.edge_edge.size();
    });
}

int ref_inclusion_box(uint8_t kind, const double* points, const double* box, double* out)
{
    return guard([&] {
        IntervalBox b;
        b.t = { box[0], box[1] };
        b.u = { box[2], box[3] };
        b.v = { box[4], box[5] };
        const IntervalVec3 r = inclusion_box(make_query(kind, points), b);
        for (int c = 0; c < 3; ++c) {
            out[2 * c] = r[c].lo;
            out[2 * c + 1] = r[c].hi;
        }
    });
}

int ref_process_interval(uint8_t kind, const double* points, const double* box,
                         const uint16_t* depth, double t_star, double sep,
                         const ccdk_narrow_cfg* cfg, uint8_t* action, double* cand_t,
                         uint8_t* zdiag, double* children, uint16_t* child_depth)
{
    return guard([&] {
        IntervalBox b;
        b.t = { box[0], box[1] };
        b.u = { box[2], box[3] };
        b.v = { box[4], box[5] };
        b.depth = { depth[0], depth[1], depth[2] };
        const ProcessResult r
            = process_interval(b, t_star, make_ncfg(cfg), make_query(kind, points), sep);
        *action = static_cast<uint8_t>(r.action);
        *cand_t = r.candidate_t;
        *zdiag = r.zero_toi_diagnostic;
        for (int ch = 0; ch < 2; ++ch) {
            const IntervalBox& c = r.children[ch];
            const double v[6] = { c.t.lo, c.t.hi, c.u.lo, c.u.hi, c.v.lo, c.v.hi };
            std::memcpy(children + 6 * ch, v, sizeof v);
            for (int d = 0; d < 3; ++d)
                child_depth[3 * ch + d] = c.depth[d];
        }
    });
}

int ref_narrow_phase(const uint8_t* kind, const double* points, uint64_t n,
                     const double* seps, const ccdk_narrow_cfg* cfg, unsigned threads,
                     uint64_t capacity, double* toi, uint8_t* flags,
                     ccdk_narrow_stats* stats)
{
    return guard([&] {
        std::vector<NarrowQuery> qs(n);
        for (uint64_t i = 0; i < n; ++i)
            qs[i] = make_query(kind[i], points + 24 * i);
        std::vector<double> sv;
        if (seps)
            sv.assign(seps, seps + n);
        const NarrowOutcome o = narrow_phase(qs, make_ncfg(cfg), threads,
                                             static_cast<size_t>(capacity),
                                             seps ? &sv : nullptr);
        for (uint64_t i = 0; i < n; ++i) {
            toi[i] = o.per_query[i].toi;
            flags[i] = (o.per_query[i].tolerance_hit ? CCDK_FLAG_TOLERANCE_HIT : 0u)
                | (o.per_query[i].zero_toi_diagnostic ? CCDK_FLAG_ZERO_TOI_DIAG : 0u);
        }
        std::memset(stats, 0, sizeof *stats);
        stats->global_toi = o.global_toi;
        stats->overflow = o.overflow;
        stats->peak_queue = o.peak_queue;
        stats->total_splits = o.total_splits;
    });
}

int ref_query_min_separations(const uint8_t* kind, const double* points, uint64_t n,
                              const ccdk_pipeline_cfg* cfg, double* out)
{
    return guard([&] {
        std::vector<NarrowQuery> qs(n);
        for (uint64_t i = 0; i < n; ++i)
            qs[i] = make_query(kind[i], points + 24 * i);
        const std::vector<double> s = query_min_separations(qs, make_pcfg(cfg));
        std::copy(s.begin(), s.end(), out);
    });
}

int ref_ccd(const double* v0, const double* v1, uint64_t nv, const uint32_t* e, uint64_t ne,
            const uint32_t* f, uint64_t nf, const ccdk_pipeline_cfg* cfg, int no_zero_retry,
            ccdk_report* rep, uint64_t** pairs)
{
    return guard([&] {
        const SceneStep s = make_scene(v0, v1, nv, e, ne, f, nf);
        const PipelineConfig pc = make_pcfg(cfg);
        const CcdReport r = no_zero_retry ? ccd_no_zero_toi(s, pc) : ccd(s, pc);
        std::memset(rep, 0, sizeof *rep);
        rep->toi = r.toi.toi;
        rep->tolerance_hit = r.toi.tolerance_hit;
        rep->zero_toi_diagnostic = r.toi.zero_toi_diagnostic;
        rep->candidate_count = r.candidate_count;
        rep->query_count = r.query_count;
        rep->batch_count = r.batch_count;
        const auto get = [&](const char* key) {
            const auto it = r.per_stage_times.find(key);
            return it == r.per_stage_times.end() ? 0.0 : it->second;
        };
        rep->t_cb = get("CB");
        rep->t_bp = get("BP");
        rep->t_socd = get("SO/CD");
        rep->t_np = get("NP");
        rep->tracked_peak_bytes = r.tracked_peak_bytes;
        if (pairs) {
            std::vector<uint64_t> flat;
            flat.reserve(2 * r.candidates.size());
            for (const auto& p : r.candidates) {
                flat.push_back(pack_id(p.left));
                flat.push_back(pack_id(p.right));
            }
            *pairs = dup(flat);
        }
    });
}

// run_batched (pipeline.cpp:179-215) on a caller's box list; the trace's
// counters go to broad_batches / narrow_batches.
int ref_run_batched(const double* v0, const double* v1, uint64_t nv, const uint32_t* e, uint64_t ne,
                    const uint32_t* f, uint64_t nf, const float* mn, const float* mx, const uint8_t* kind,
                    const uint32_t* index, uint64_t k, const ccdk_pipeline_cfg* cfg, ccdk_report* rep,
                    uint64_t* broad_batches, uint64_t* narrow_batches, uint64_t** pairs)
{
    return guard([&] {
        const SceneStep s = make_scene(v0, v1, nv, e, ne, f, nf);
        const std::vector<Aabb> boxes = make_boxes(mn, mx, kind, index, k);
        const PipelineConfig pc = make_pcfg(cfg);
        BatchTrace trace;
        CcdReport r;
        const ToiResult t = run_batched(s, boxes, pc, trace, &r);
        std::memset(rep, 0, sizeof *rep);
        rep->toi = t.toi;
        rep->tolerance_hit = t.tolerance_hit;
        rep->zero_toi_diagnostic = t.zero_toi_diagnostic;
        rep->candidate_count = r.candidate_count;
        rep->query_count = r.query_count;
        rep->batch_count = r.batch_count;
        rep->tracked_peak_bytes = r.tracked_peak_bytes;
        *broad_batches = trace.broad_batches;
        *narrow_batches = trace.narrow_batches;
        std::vector<uint64_t> flat;
        flat.reserve(2 * r.candidates.size());
        for (const auto& p : r.candidates) {
            flat.push_back(pack_id(p.left));
            flat.push_back(pack_id(p.right));
        }
        *pairs = dup(flat);
    });
}

int ref_make_cloth_scene(uint64_t nx, uint64_t ny, double jitter, double drop,
                         uint64_t seed, double** v0, double** v1, uint64_t* nv,
                         uint32_t** e, uint64_t* ne, uint32_t** f, uint64_t* nf)
{
    return guard([&] {
        scene_out(make_cloth_scene(nx, ny, jitter, drop, seed), v0, v1, nv, e, ne, f, nf);
    });
}

int ref_make_box_soup(uint64_t count, double region, double size, double motion,
                      uint64_t seed, double** v0, double** v1, uint64_t* nv,
                      uint32_t** e, uint64_t* ne, uint32_t** f, uint64_t* nf)
{
    return guard([&] {
        scene_out(make_box_soup(count, region, size, motion, seed), v0, v1, nv, e, ne, f,
                  nf);
    });
}

int ref_distances(const uint8_t* kind, const double* points, uint64_t n, double* out)
{
    return guard([&] {
        for (uint64_t i = 0; i < n; ++i) {
            const NarrowQuery q = make_query(kind[i], points + 24 * i);
            out[i] = kind[i] ? segment_segment_distance(q.points_t0[0], q.points_t0[1],
                                                        q.points_t0[2], q.points_t0[3])
                             : point_triangle_distance(q.points_t0[0], q.points_t0[1],
                                                       q.points_t0[2], q.points_t0[3]);
        }
    });
}

} // extern "C"
