// Reference-style tests for the C++ drop-in API (include/ccdkit/*.hpp over
// libccdkit.so -> libccdk.so).  Re-authored from the reference's doctest
// suites (proj/tests/test_{geometry,broadphase,narrowphase,pipeline}.cpp) with
// a minimal harness; built and run by tests/test_cpp_api.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "ccdkit/aabb.hpp"
#include "ccdkit/broadphase.hpp"
#include "ccdkit/distance.hpp"
#include "ccdkit/narrowphase.hpp"
#include "ccdkit/pipeline.hpp"

using namespace ccdkit;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                       \
    do {                                                                                  \
        ++g_checks;                                                                       \
        if (!(cond)) {                                                                    \
            ++g_fail;                                                                     \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);                    \
        }                                                                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                          \
    do {                                                                                  \
        ++g_checks;                                                                       \
        bool ok__ = false;                                                                \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const T&) {                                                              \
            ok__ = true;                                                                  \
        } catch (...) {                                                                   \
        }                                                                                 \
        if (!ok__) {                                                                      \
            ++g_fail;                                                                     \
            std::printf("FAIL %s:%d %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
        }                                                                                 \
    } while (0)

static SceneStep plane_scene()
{
    SceneStep s;
    s.vertices_t0 = { { 0, 0, 0 }, { 1, 0, 0 }, { 0, 1, 0 }, { 0.25, 0.25, 1 } };
    s.vertices_t1 = { { 0, 0, 0 }, { 1, 0, 0 }, { 0, 1, 0 }, { 0.25, 0.25, -1 } };
    s.faces = { { 0, 1, 2 } };
    s.edges = { { 0, 1 }, { 0, 2 }, { 1, 2 } };
    return s;
}

static NarrowQuery plane_query()
{
    NarrowQuery q;
    q.points_t0 = { Vec3 { 0.25, 0.25, 1 }, { 0, 0, 0 }, { 1, 0, 0 }, { 0, 1, 0 } };
    q.points_t1 = { Vec3 { 0.25, 0.25, -1 }, { 0, 0, 0 }, { 1, 0, 0 }, { 0, 1, 0 } };
    return q;
}

static void geometry()
{
    CHECK(round_down_reduced(1.0) == 1.0f && round_up_reduced(-2.5) == -2.5f);
    CHECK(round_down_reduced(0.1) == std::nextafterf(static_cast<float>(0.1), -1.0f));
    CHECK(round_up_reduced(0.1) == static_cast<float>(0.1));
    CHECK_THROWS_AS(round_down_reduced(std::nan("")), InvalidInput);
    SceneStep e;
    e.vertices_t0 = { { 0, 0, 0 }, { 1, 0, 0 } };
    e.vertices_t1 = { { 0, 0, 1 }, { 1, 0, 1 } };
    e.edges = { { 0, 1 } };
    const auto boxes = build_boxes(e);
    CHECK(boxes.size() == 3);
    CHECK(boxes[2].owner == (PrimitiveId { PrimitiveKind::Edge, 0 }));
    CHECK((boxes[2].max_corner == std::array<float, 3> { 1, 0, 1 }));
    SceneStep bad = e;
    bad.edges = { { 0, 0 } };
    CHECK_THROWS_AS(build_boxes(bad), InvalidInput);
}

static void broadphase()
{
    const SceneStep s = plane_scene();
    const auto boxes = build_boxes(s, 0.01);
    StqStats stats;
    const auto a = stq(boxes, s, 1, &stats);
    CHECK(a == sap(boxes, s) && a == bf(boxes, s));
    CHECK(stats.max_queue <= boxes.size() - 1);
    const auto vf = make_pair_canonical({ PrimitiveKind::Face, 0 }, { PrimitiveKind::Vertex, 3 });
    CHECK(std::find(a.begin(), a.end(), vf) != a.end());
    const ClassifiedQueries q = classify({ vf }, s);
    CHECK(q.vertex_face.size() == 1 && q.edge_edge.empty());
    CHECK(q.vertex_face[0].points_t0[0] == s.vertices_t0[3]);
    CHECK(q.vertex_face[0].source == vf);
    CHECK_THROWS_AS(classify({ make_pair_canonical({ PrimitiveKind::Vertex, 0 }, { PrimitiveKind::Face, 9 }) }, s),
                    InvalidInput);
    CHECK_THROWS_AS(choose_axis({}), InvalidInput);
}

static void narrowphase()
{
    const NarrowQuery q = plane_query();
    const IntervalVec3 b = inclusion_box(q, IntervalBox {});
    CHECK(b.z.lo <= -1.0 && b.z.hi >= 1.0);
    IntervalBox late;
    late.t = { 0.5, 1.0 };
    late.depth[0] = 1;
    CHECK(process_interval(late, 0.25, NarrowConfig {}, q).action == IntervalAction::Pruned);
    const NarrowOutcome one = narrow_phase({ q }, NarrowConfig {});
    CHECK(one.per_query.size() == 1);
    CHECK(one.global_toi == 0.5 - std::ldexp(1.0, -21));
    CHECK(one.total_splits == 449 && one.peak_queue == 16);
    CHECK(narrow_phase({ q, q, q }, NarrowConfig {}, 1, 2).overflow);
    NarrowConfig four;
    four.max_splits = 4;
    const NarrowOutcome ex = narrow_phase({ q }, four);
    CHECK(ex.per_query[0].tolerance_hit && ex.per_query[0].toi == 0.25);
    NarrowConfig sep;
    sep.min_separation = 0.25;
    CHECK(narrow_phase({ q }, sep).global_toi == 0.37451171875);
    NarrowConfig bad;
    bad.delta = 0.0;
    CHECK_THROWS_AS(narrow_phase({ q }, bad), ConfigError);
    IntervalBox l, r;
    split_box(IntervalBox {}, 0, l, r);
    CHECK(l.t.hi == 0.5 && r.t.lo == 0.5 && l.depth[0] == 1);
}

static void pipeline()
{
    const SceneStep s = plane_scene();
    const CcdReport r = ccd(s, PipelineConfig {});
    CHECK(r.toi.collision() && r.toi.toi <= 0.5 && r.toi.toi >= 0.5 - std::ldexp(1.0, -20));
    CHECK(r.per_stage_times.count("CB") && r.per_stage_times.count("NP"));
    PipelineConfig tiny;
    tiny.memory_budget = 100;
    CHECK_THROWS_AS(ccd(s, tiny), ConfigError);
    PipelineConfig rel;
    rel.min_sep_mode = MinSepMode::Relative;
    const auto cq = classify({ make_pair_canonical({ PrimitiveKind::Vertex, 3 }, { PrimitiveKind::Face, 0 }) }, s);
    const auto seps = query_min_separations(cq.vertex_face, rel);
    CHECK(seps.size() == 1 && seps[0] == 0.2 * 1.0);
    CHECK(point_triangle_distance(s.vertices_t0[3], s.vertices_t0[0], s.vertices_t0[1], s.vertices_t0[2]) == 1.0);
    PipelineConfig nz;
    CHECK_THROWS_AS(ccd_no_zero_toi(s, nz), ConfigError);
    SceneStep hover = s;
    hover.vertices_t0[3] = { 0.25, 0.25, 1e-13 };
    nz.narrow.no_zero_toi = true;
    nz.narrow.min_separation = 1e-6;
    const CcdReport z = ccd_no_zero_toi(hover, nz);
    PipelineConfig retry = nz;
    retry.narrow.min_separation = 0.0;
    CHECK(z.toi.toi == kZeroToiRetryScale * ccd(hover, retry).toi.toi);
    BatchTrace trace;
    CcdReport rb;
    const ToiResult t = run_batched(s, build_boxes(s), PipelineConfig {}, trace, &rb);
    CHECK(t.toi == r.toi.toi && trace.narrow_batches == 1);
}

// A grid of n x n vertices falling through z = 0 with a slight tilt.
static SceneStep grid_scene(int n, double tilt)
{
    SceneStep s;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            s.vertices_t0.push_back({ double(i), double(j), 1.0 + tilt * i });
            s.vertices_t1.push_back({ double(i) + 0.1, double(j), -1.0 + tilt * j });
        }
    for (int j = 0; j + 1 < n; ++j)
        for (int i = 0; i + 1 < n; ++i) {
            const uint32_t a = j * n + i, b = a + 1, c = a + n, d = c + 1;
            s.faces.push_back({ a, b, d });
            s.faces.push_back({ a, d, c });
            s.edges.push_back({ a, b });
            s.edges.push_back({ a, c });
            s.edges.push_back({ a, d });
        }
    for (int j = 0; j + 1 < n; ++j)
        s.edges.push_back({ uint32_t(j * n + n - 1), uint32_t((j + 1) * n + n - 1) });
    for (int i = 0; i + 1 < n; ++i)
        s.edges.push_back({ uint32_t((n - 1) * n + i), uint32_t((n - 1) * n + i + 1) });
    // a static floor triangle under the grid
    const uint32_t f = uint32_t(s.vertices_t0.size());
    for (const Vec3& v : { Vec3 { -1, -1, 0 }, Vec3 { 3.0 * n, -1, 0 }, Vec3 { -1, 3.0 * n, 0 } }) {
        s.vertices_t0.push_back(v);
        s.vertices_t1.push_back(v);
    }
    s.faces.push_back({ f, f + 1, f + 2 });
    s.edges.push_back({ f, f + 1 });
    s.edges.push_back({ f, f + 2 });
    s.edges.push_back({ f + 1, f + 2 });
    return s;
}

// Reentrancy (test_pipeline.cpp:96-106, test_narrowphase.cpp:196-211): calls
// from several threads, with any `threads` value, return the single-threaded
// results, candidate lists included.
static void determinism_across_threads()
{
    const SceneStep a = grid_scene(12, 0.01), b = grid_scene(9, -0.02);
    const CcdReport ra = ccd(a, PipelineConfig {}), rb = ccd(b, PipelineConfig {});
    CHECK(!ra.candidates.empty() && ra.candidates.size() != rb.candidates.size());
    const auto boxes = build_boxes(b);
    const auto pairs = stq(boxes, b);
    const auto q = classify(pairs, b);
    const NarrowOutcome nb = narrow_phase(q.vertex_face, NarrowConfig {});
    std::vector<int> bad(4, 0);
    std::vector<std::thread> ts;
    for (int t = 0; t < 4; ++t)
        ts.emplace_back([&, t] {
            for (int it = 0; it < 6; ++it) {
                const int k = (t + it) % 3;
                if (k == 0) {
                    const CcdReport r = ccd(t % 2 ? b : a, PipelineConfig {});
                    const CcdReport& e = t % 2 ? rb : ra;
                    bad[t] += !(r.candidates == e.candidates && r.toi.toi == e.toi.toi);
                } else if (k == 1) {
                    bad[t] += !(stq(boxes, b, 1 + 7 * (t % 2)) == pairs);
                } else {
                    const NarrowOutcome o = narrow_phase(q.vertex_face, NarrowConfig {}, 8);
                    bool same = o.total_splits == nb.total_splits && o.per_query.size() == nb.per_query.size();
                    for (size_t i = 0; same && i < o.per_query.size(); ++i)
                        same = o.per_query[i].toi == nb.per_query[i].toi;
                    bad[t] += !same;
                }
            }
        });
    for (auto& th : ts)
        th.join();
    for (int t = 0; t < 4; ++t)
        CHECK(bad[t] == 0);
}

// run_batched on a caller's box list (pipeline.cpp:179-215): reversed order,
// padded boxes and a duplicated owner sweep like any other list; the report
// keeps the fields run_batched does not write (CB); the trace accumulates.
static void run_batched_on_a_box_list()
{
    const SceneStep s = grid_scene(10, 0.01);
    std::vector<Aabb> boxes = build_boxes(s, 0.0);
    std::reverse(boxes.begin(), boxes.end());
    for (Aabb& b : boxes)
        for (int c = 0; c < 3; ++c) {
            b.min_corner[c] -= 0.05f;
            b.max_corner[c] += 0.05f;
        }
    boxes.push_back(boxes.front());
    // the expected list: the broad phase on the same boxes + classify/narrow
    const auto pairs = stq(boxes, s);
    const ClassifiedQueries q = classify(pairs, s);
    std::vector<NarrowQuery> all = q.vertex_face;
    all.insert(all.end(), q.edge_edge.begin(), q.edge_edge.end());
    const NarrowOutcome o = narrow_phase(all, NarrowConfig {});
    BatchTrace trace;
    CcdReport rep;
    rep.per_stage_times["CB"] = 0.25;
    const ToiResult t = run_batched(s, boxes, PipelineConfig {}, trace, &rep);
    CHECK(rep.candidates == pairs);
    CHECK(t.toi == o.global_toi && rep.toi.toi == t.toi);
    CHECK(rep.query_count == all.size() && trace.broad_batches == 1 && trace.narrow_batches == 1);
    CHECK(rep.per_stage_times["CB"] == 0.25);
    // a small budget: several broad batches.  Each batch is deduplicated on
    // its own and the union is only sorted (pipeline.cpp:196), so the
    // duplicated owner can repeat a pair across batches, as in the reference
    PipelineConfig small;
    small.memory_budget = 1 << 15;
    CcdReport rs;
    const ToiResult ts = run_batched(s, boxes, small, trace, &rs);
    std::vector<CandidatePair> uniq = rs.candidates;
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    CHECK(ts.toi == t.toi && uniq == pairs && std::is_sorted(rs.candidates.begin(), rs.candidates.end()));
    CHECK(trace.broad_batches > 2);
    CHECK(rs.batch_count == trace.narrow_batches);
    std::printf("run_batched: %zu candidates, budget 2^15: trace %zu broad / %zu narrow batches\n", pairs.size(),
                trace.broad_batches, trace.narrow_batches);
    // owners must name existing primitives
    std::vector<Aabb> bad = boxes;
    bad[0].owner.index = 1u << 30;
    CHECK_THROWS_AS(run_batched(s, bad, PipelineConfig {}, trace, nullptr), InvalidInput);
}

int main()
{
    try {
        geometry();
        broadphase();
        narrowphase();
        pipeline();
        determinism_across_threads();
        run_batched_on_a_box_list();
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
