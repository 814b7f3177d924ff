// The reference's C++ API (include/ccdkit/*.hpp) implemented over the C ABI
// (include/ccdk.h): link against libccdkit.so instead of the reference's
// libccdkit.a and every hot-path call runs on the B200.
//
// The shim only converts containers and maps status codes to the reference's
// exceptions (InvalidInput / ConfigError); all compute is a ccdk_* call.
// Scene validation and share_vertex are data-model helpers of SceneStep and
// run on the host, as the reference's do.  One process-wide device context
// (CCDK_DEVICE, default 0) serves all calls; the C ABI serialises them, and
// calls that produce a result and then fetch it from the context (ccd,
// stq/bf/sap, run_batched) hold the shim's lock across both, so the API is
// reentrant like the reference's (SURVEY §8(b) threading).
#include "ccdkit/aabb.hpp"
#include "ccdkit/broadphase.hpp"
#include "ccdkit/distance.hpp"
#include "ccdkit/narrowphase.hpp"
#include "ccdkit/pipeline.hpp"
#include "ccdkit/scene.hpp"

#include <sys/mman.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>
#include <mutex>
#include <stdexcept>

#include "ccdk.h"

#define CCDKIT_EXPORT __attribute__((visibility("default")))

namespace ccdkit {

namespace {

// held across a produce-then-fetch sequence on the shared context
std::recursive_mutex& sequence_mutex()
{
    static std::recursive_mutex m;
    return m;
}
using SequenceGuard = std::lock_guard<std::recursive_mutex>;

ccdk_ctx* context()
{
    static std::once_flag once;
    static ccdk_ctx* ctx = nullptr;
    static int rc = 0;
    std::call_once(once, [] {
        const char* d = std::getenv("CCDK_DEVICE");
        rc = ccdk_ctx_create(d ? std::atoi(d) : 0, &ctx);
    });
    if (rc != CCDK_OK)
        throw std::runtime_error(std::string("ccdkit: no CUDA device context: ") + ccdk_last_error());
    return ctx;
}

void check(int rc)
{
    if (rc == CCDK_OK)
        return;
    const std::string msg = ccdk_last_error();
    if (rc == CCDK_INVALID_INPUT)
        throw InvalidInput(msg);
    if (rc == CCDK_CONFIG)
        throw ConfigError(msg);
    throw std::runtime_error("ccdk: " + msg);
}

const double* vdata(const std::vector<Vec3>& v) { return v.empty() ? nullptr : v[0].data(); }
const uint32_t* edata(const SceneStep& s) { return s.edges.empty() ? nullptr : s.edges[0].data(); }
const uint32_t* fdata(const SceneStep& s) { return s.faces.empty() ? nullptr : s.faces[0].data(); }

uint64_t pack(PrimitiveId id) { return (uint64_t(id.kind) << 32) | id.index; }
PrimitiveId unpack(uint64_t v) { return { PrimitiveKind(v >> 32), uint32_t(v) }; }

ccdk_narrow_cfg to_c(const NarrowConfig& n)
{
    ccdk_narrow_cfg c {};
    c.delta = n.delta;
    c.min_separation = n.min_separation;
    c.t_max = n.t_max;
    c.max_splits = n.max_splits;
    c.no_zero_toi = n.no_zero_toi ? 1 : 0;
    return c;
}

ccdk_pipeline_cfg to_c(const PipelineConfig& p)
{
    ccdk_pipeline_cfg c {};
    c.narrow = to_c(p.narrow);
    c.broad_method = int32_t(p.broad_method);
    c.min_sep_mode = int32_t(p.min_sep_mode);
    c.memory_budget = p.memory_budget;
    c.rs_params = p.record_sizes.params;
    c.rs_query = p.record_sizes.query;
    c.rs_interval = p.record_sizes.interval;
    c.rs_pair_ints = p.record_sizes.pair_ints;
    c.min_sep_fraction = p.min_sep_fraction;
    c.threads = p.threads;
    c.inflation = p.inflation;
    return c;
}

void flatten(const NarrowQuery& q, uint8_t& kind, double* p)
{
    kind = q.kind == QueryKind::EdgeEdge ? CCDK_QUERY_EE : CCDK_QUERY_VF;
    for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) {
            p[3 * i + c] = q.points_t0[i][c];
            p[12 + 3 * i + c] = q.points_t1[i][c];
        }
}

NarrowQuery unflatten(uint8_t kind, const double* p, uint64_t left, uint64_t right)
{
    NarrowQuery q;
    q.kind = kind == CCDK_QUERY_EE ? QueryKind::EdgeEdge : QueryKind::VertexFace;
    for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) {
            q.points_t0[i][c] = p[3 * i + c];
            q.points_t1[i][c] = p[12 + 3 * i + c];
        }
    q.source = { unpack(left), unpack(right) };
    return q;
}

std::vector<CandidatePair> fetch_pairs(uint64_t n)
{
    std::vector<uint64_t> flat(2 * n);
    if (n)
        check(ccdk_fetch_pairs(context(), flat.data()));
    std::vector<CandidatePair> out(n);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = { unpack(flat[2 * i]), unpack(flat[2 * i + 1]) };
    return out;
}

// A box list as the C ABI takes it: corners [k][3], owner kinds, indices.
struct BoxArrays {
    std::vector<float> mn, mx;
    std::vector<uint8_t> kind;
    std::vector<uint32_t> index;
    explicit BoxArrays(const std::vector<Aabb>& boxes)
        : mn(3 * boxes.size()), mx(3 * boxes.size()), kind(boxes.size()), index(boxes.size())
    {
        for (size_t i = 0; i < boxes.size(); ++i) {
            for (int c = 0; c < 3; ++c) {
                mn[3 * i + c] = boxes[i].min_corner[c];
                mx[3 * i + c] = boxes[i].max_corner[c];
            }
            kind[i] = uint8_t(boxes[i].owner.kind);
            index[i] = boxes[i].owner.index;
        }
    }
};

std::vector<CandidatePair> broad(int method, const std::vector<Aabb>& boxes, const SceneStep& scene,
                                 StqStats* stats, SweepRange range)
{
    SequenceGuard g(sequence_mutex());
    const size_t k = boxes.size();
    const BoxArrays b(boxes);
    uint64_t n = 0;
    ccdk_stq_stats st {};
    check(ccdk_broad_phase(context(), method, b.mn.data(), b.mx.data(), b.kind.data(), b.index.data(), k,
                           scene.vertices_t0.size(), edata(scene), scene.edges.size(), fdata(scene),
                           scene.faces.size(), range.begin, range.end, &n, stats ? &st : nullptr));
    std::vector<CandidatePair> out = fetch_pairs(n);
    if (stats) {
        std::vector<uint64_t> rounds(st.n_rounds);
        if (st.n_rounds)
            check(ccdk_fetch_round_sizes(context(), rounds.data()));
        for (uint64_t r : rounds)
            stats->round_sizes.push_back(size_t(r));
        stats->max_queue = std::max<size_t>(stats->max_queue, size_t(st.max_queue));
    }
    return out;
}

CcdReport to_report(const ccdk_report& r, bool with_candidates)
{
    CcdReport rep;
    rep.toi = { r.toi, r.tolerance_hit != 0, r.zero_toi_diagnostic != 0 };
    rep.candidate_count = r.candidate_count;
    rep.query_count = r.query_count;
    rep.batch_count = r.batch_count;
    rep.per_stage_times["CB"] = r.t_cb;
    rep.per_stage_times["BP"] = r.t_bp;
    rep.per_stage_times["SO/CD"] = r.t_socd;
    rep.per_stage_times["NP"] = r.t_np;
    rep.tracked_peak_bytes = r.tracked_peak_bytes;
    if (with_candidates)
        rep.candidates = fetch_pairs(r.candidate_count);
    // the API's own record sizes, as the reference reports them
    // (pipeline.cpp:210-213); the device layouts are internal
    rep.real_record_sizes.params = sizeof(PipelineConfig);
    rep.real_record_sizes.query = sizeof(NarrowQuery);
    rep.real_record_sizes.interval = sizeof(IntervalBox) + sizeof(ProcessResult);
    rep.real_record_sizes.pair_ints = sizeof(CandidatePair);
    return rep;
}

} // namespace

// ------------------------------------------------------------------ scene

CCDKIT_EXPORT void SceneStep::validate() const
{
    if (vertices_t0.size() != vertices_t1.size())
        throw InvalidInput("vertex snapshots differ in length");
    const size_t n = vertices_t0.size();
    for (size_t i = 0; i < n; ++i)
        if (!is_finite(vertices_t0[i]) || !is_finite(vertices_t1[i]))
            throw InvalidInput("non-finite vertex coordinate");
    for (const auto& e : edges) {
        if (e[0] >= n || e[1] >= n)
            throw InvalidInput("edge index out of range");
        if (e[0] == e[1])
            throw InvalidInput("edge endpoints must be distinct");
    }
    for (const auto& f : faces) {
        if (f[0] >= n || f[1] >= n || f[2] >= n)
            throw InvalidInput("face index out of range");
        if (f[0] == f[1] || f[1] == f[2] || f[0] == f[2])
            throw InvalidInput("face vertices must be distinct");
    }
}

static int vertices_of(const SceneStep& s, PrimitiveId id, std::array<uint32_t, 3>& out)
{
    switch (id.kind) {
    case PrimitiveKind::Vertex:
        out[0] = id.index;
        return 1;
    case PrimitiveKind::Edge:
        out[0] = s.edges[id.index][0];
        out[1] = s.edges[id.index][1];
        return 2;
    case PrimitiveKind::Face:
        out = s.faces[id.index];
        return 3;
    }
    return 0;
}

CCDKIT_EXPORT bool uses_vertex(const SceneStep& scene, PrimitiveId id, std::uint32_t v)
{
    std::array<uint32_t, 3> w {};
    const int n = vertices_of(scene, id, w);
    return std::find(w.begin(), w.begin() + n, v) != w.begin() + n;
}

CCDKIT_EXPORT bool share_vertex(const SceneStep& scene, PrimitiveId a, PrimitiveId b)
{
    std::array<uint32_t, 3> wa {};
    const int na = vertices_of(scene, a, wa);
    for (int i = 0; i < na; ++i)
        if (uses_vertex(scene, b, wa[i]))
            return true;
    return false;
}

// ------------------------------------------------------------------- aabb

CCDKIT_EXPORT float round_down_reduced(double x)
{
    float d, u;
    check(ccdk_round_reduced(context(), &x, 1, &d, &u));
    return d;
}

CCDKIT_EXPORT float round_up_reduced(double x)
{
    float d, u;
    check(ccdk_round_reduced(context(), &x, 1, &d, &u));
    return u;
}

CCDKIT_EXPORT std::vector<Aabb> build_boxes(const SceneStep& scene, double inflation, unsigned)
{
    if (scene.vertices_t0.size() != scene.vertices_t1.size())
        throw InvalidInput("vertex snapshots differ in length");
    const size_t k = scene.primitive_count();
    std::vector<float> mn(3 * k), mx(3 * k);
    std::vector<uint8_t> kind(k);
    std::vector<uint32_t> index(k);
    check(ccdk_build_boxes(context(), vdata(scene.vertices_t0), vdata(scene.vertices_t1),
                           scene.vertices_t0.size(), edata(scene), scene.edges.size(), fdata(scene),
                           scene.faces.size(), inflation, mn.data(), mx.data(), kind.data(),
                           index.data()));
    std::vector<Aabb> boxes(k);
    for (size_t i = 0; i < k; ++i) {
        for (int c = 0; c < 3; ++c) {
            boxes[i].min_corner[c] = mn[3 * i + c];
            boxes[i].max_corner[c] = mx[3 * i + c];
        }
        boxes[i].owner = { PrimitiveKind(kind[i]), index[i] };
    }
    return boxes;
}

// ------------------------------------------------------------- broadphase

CCDKIT_EXPORT int choose_axis(const std::vector<Aabb>& boxes)
{
    if (boxes.empty())
        throw InvalidInput("choose_axis: empty box list");
    std::vector<float> mn(3 * boxes.size()), mx(3 * boxes.size());
    for (size_t i = 0; i < boxes.size(); ++i)
        for (int c = 0; c < 3; ++c) {
            mn[3 * i + c] = boxes[i].min_corner[c];
            mx[3 * i + c] = boxes[i].max_corner[c];
        }
    int axis = 0;
    check(ccdk_choose_axis(context(), mn.data(), mx.data(), boxes.size(), &axis));
    return axis;
}

CCDKIT_EXPORT std::vector<CandidatePair> stq(const std::vector<Aabb>& boxes, const SceneStep& scene,
                                             unsigned, StqStats* stats, SweepRange range)
{
    return broad(CCDK_BROAD_STQ, boxes, scene, stats, range);
}

CCDKIT_EXPORT std::vector<CandidatePair> bf(const std::vector<Aabb>& boxes, const SceneStep& scene,
                                            unsigned, SweepRange range)
{
    return broad(CCDK_BROAD_BF, boxes, scene, nullptr, range);
}

CCDKIT_EXPORT std::vector<CandidatePair> sap(const std::vector<Aabb>& boxes, const SceneStep& scene,
                                             unsigned, SweepRange range)
{
    return broad(CCDK_BROAD_SAP, boxes, scene, nullptr, range);
}

CCDKIT_EXPORT ClassifiedQueries classify(const std::vector<CandidatePair>& pairs, const SceneStep& scene)
{
    const size_t n = pairs.size();
    ClassifiedQueries out;
    if (!n)
        return out;
    std::vector<uint64_t> flat(2 * n);
    for (size_t i = 0; i < n; ++i) {
        flat[2 * i] = pack(pairs[i].left);
        flat[2 * i + 1] = pack(pairs[i].right);
    }
    std::vector<uint8_t> kind(n);
    std::vector<double> pts(24 * n);
    std::vector<uint64_t> src(2 * n);
    uint64_t nvf = 0, nee = 0;
    check(ccdk_classify(context(), flat.data(), n, vdata(scene.vertices_t0), vdata(scene.vertices_t1),
                        scene.vertices_t0.size(), edata(scene), scene.edges.size(), fdata(scene),
                        scene.faces.size(), kind.data(), pts.data(), src.data(), &nvf, &nee));
    for (uint64_t i = 0; i < nvf + nee; ++i)
        (i < nvf ? out.vertex_face : out.edge_edge)
            .push_back(unflatten(kind[i], &pts[24 * i], src[2 * i], src[2 * i + 1]));
    return out;
}

// ------------------------------------------------------------ narrowphase

CCDKIT_EXPORT void NarrowConfig::validate() const
{
    if (!(delta > 0.0))
        throw ConfigError("NarrowConfig: delta must be > 0");
    if (max_splits < 1)
        throw ConfigError("NarrowConfig: max_splits must be >= 1");
    if (min_separation < 0.0)
        throw ConfigError("NarrowConfig: min_separation must be >= 0");
    if (!(t_max > 0.0) || t_max > 1.0)
        throw ConfigError("NarrowConfig: t_max must be in (0, 1]");
}

CCDKIT_EXPORT IntervalVec3 inclusion_box(const NarrowQuery& query, const IntervalBox& box)
{
    uint8_t kind;
    double pts[24];
    flatten(query, kind, pts);
    const double b[6] = { box.t.lo, box.t.hi, box.u.lo, box.u.hi, box.v.lo, box.v.hi };
    double out[6];
    check(ccdk_inclusion_boxes(context(), &kind, pts, b, 1, out));
    return { { out[0], out[1] }, { out[2], out[3] }, { out[4], out[5] } };
}

CCDKIT_EXPORT ProcessResult process_interval(const IntervalBox& box, double t_star,
                                             const NarrowConfig& cfg, const NarrowQuery& query,
                                             double min_separation)
{
    uint8_t kind, action, zd;
    double pts[24], cand, children[12];
    uint16_t child_depth[6];
    flatten(query, kind, pts);
    const double b[6] = { box.t.lo, box.t.hi, box.u.lo, box.u.hi, box.v.lo, box.v.hi };
    const ccdk_narrow_cfg c = to_c(cfg);
    check(ccdk_process_intervals(context(), &kind, pts, b, box.depth.data(), &t_star, &min_separation, 1,
                                 &c, &action, &cand, &zd, children, child_depth));
    ProcessResult r;
    r.action = IntervalAction(action);
    r.candidate_t = cand;
    r.zero_toi_diagnostic = zd != 0;
    if (r.action == IntervalAction::Split)
        for (int s = 0; s < 2; ++s) {
            IntervalBox& ch = r.children[s];
            ch.query_id = box.query_id;
            ch.t = { children[6 * s], children[6 * s + 1] };
            ch.u = { children[6 * s + 2], children[6 * s + 3] };
            ch.v = { children[6 * s + 4], children[6 * s + 5] };
            ch.depth = { child_depth[3 * s], child_depth[3 * s + 1], child_depth[3 * s + 2] };
        }
    return r;
}

CCDKIT_EXPORT void split_box(const IntervalBox& box, int d, IntervalBox& left, IntervalBox& right)
{
    // exact dyadic bisection: index bookkeeping, kept on the host like the
    // reference's inline helper (narrowphase.cpp:122-132)
    const DomainInterval& iv = box.dim(d);
    const double mid = iv.lo + 0.5 * (iv.hi - iv.lo);
    left = box;
    right = box;
    left.dim(d).hi = mid;
    right.dim(d).lo = mid;
    ++left.depth[d];
    ++right.depth[d];
}

CCDKIT_EXPORT NarrowOutcome narrow_phase(const std::vector<NarrowQuery>& queries,
                                         const NarrowConfig& cfg, unsigned, std::size_t queue_capacity,
                                         const std::vector<double>* per_query_min_sep)
{
    cfg.validate();
    const size_t n = queries.size();
    if (per_query_min_sep && per_query_min_sep->size() != n)
        throw ConfigError("narrow_phase: per-query separation list size mismatch");
    NarrowOutcome out;
    out.per_query.assign(n, ToiResult {});
    if (!n)
        return out;
    std::vector<uint8_t> kind(n), flags(n);
    std::vector<double> pts(24 * n), toi(n);
    for (size_t i = 0; i < n; ++i)
        flatten(queries[i], kind[i], &pts[24 * i]);
    const ccdk_narrow_cfg c = to_c(cfg);
    ccdk_narrow_stats st {};
    check(ccdk_narrow_phase(context(), kind.data(), pts.data(),
                            per_query_min_sep ? per_query_min_sep->data() : nullptr, n, &c,
                            queue_capacity, toi.data(), flags.data(), &st));
    for (size_t i = 0; i < n; ++i)
        out.per_query[i] = { toi[i], (flags[i] & CCDK_FLAG_TOLERANCE_HIT) != 0,
                             (flags[i] & CCDK_FLAG_ZERO_TOI_DIAG) != 0 };
    out.global_toi = st.global_toi;
    out.overflow = st.overflow != 0;
    out.peak_queue = st.peak_queue;
    out.total_splits = st.total_splits;
    return out;
}

// --------------------------------------------------------------- pipeline

CCDKIT_EXPORT const char* to_string(BroadMethod m)
{
    switch (m) {
    case BroadMethod::STQ:
        return "stq";
    case BroadMethod::BF:
        return "bf";
    case BroadMethod::SAP:
        return "sap";
    }
    return "?";
}

CCDKIT_EXPORT void PipelineConfig::validate() const
{
    narrow.validate();
    if (!record_sizes.params || !record_sizes.query || !record_sizes.interval || !record_sizes.pair_ints)
        throw ConfigError("PipelineConfig: record sizes must be positive");
    if (memory_budget <= record_sizes.params)
        throw ConfigError("PipelineConfig: memory budget must exceed the parameter size");
    if (min_sep_fraction < 0.0)
        throw ConfigError("PipelineConfig: min_sep_fraction must be >= 0");
    if (threads < 1)
        throw ConfigError("PipelineConfig: threads must be >= 1");
    if (inflation < 0.0)
        throw ConfigError("PipelineConfig: inflation must be >= 0");
}

// ccdk_ccd_into's sink: the pinned pair list is in CandidatePair's own layout
// ({u8 kind, pad, u32 index} x 2), so the report's vector is filled by one
// copy — on the library's worker thread, while the device runs the narrow
// phase.
static_assert(sizeof(PrimitiveId) == 8 && offsetof(PrimitiveId, index) == 4 && sizeof(CandidatePair) == 16
                  && offsetof(CandidatePair, right) == 8,
              "CandidatePair layout differs from the ccdk_pairs_sink contract");

namespace {

#ifdef MADV_POPULATE_WRITE
constexpr int kPopulateWrite = MADV_POPULATE_WRITE;
#else
constexpr int kPopulateWrite = 23; // Linux 5.14+; older kernels reject it (EINVAL): a no-op hint
#endif

struct CandidateSink {
    std::vector<CandidatePair>* out;
    std::exception_ptr err;
};

// Fault in a fresh destination before the copy: 2 MB pages where the kernel
// allows them (transparent huge pages in madvise mode) and the page tables
// populated by several threads at once.  A 2M-candidate list is 34 MB; faulted
// 4 KB at a time by the copy itself it costs more host time than the whole
// device step.  Hints only: any failure leaves the ordinary fault path.
void prefault(void* p, size_t bytes)
{
    constexpr uintptr_t kPage = 4096, kHuge = uintptr_t(2) << 20;
    if (bytes < 4 * kHuge)
        return;
    const uintptr_t b = (reinterpret_cast<uintptr_t>(p) + kPage - 1) & ~(kPage - 1);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(kPage - 1);
    madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = static_cast<unsigned>(std::min<uintptr_t>({ 4u, std::max(1u, hw / 2), (e - b) / kHuge }));
    const uintptr_t chunk = ((e - b) / nt + kHuge - 1) & ~(kHuge - 1);
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) {
        const uintptr_t s = b + t * chunk, f = std::min(e, s + chunk);
        if (s < f)
            pool.emplace_back([s, f] { madvise(reinterpret_cast<void*>(s), f - s, kPopulateWrite); });
    }
    madvise(reinterpret_cast<void*>(b), std::min(e, b + chunk) - b, kPopulateWrite);
    for (auto& th : pool)
        th.join();
}

int candidate_sink(void* user, const uint64_t* pairs, uint64_t n)
{
    auto* st = static_cast<CandidateSink*>(user);
    try {
        if (!pairs) { // the count, while the copy is in flight: allocate and fault in
            st->out->clear();
            st->out->reserve(n);
            prefault(st->out->data(), n * sizeof(CandidatePair));
            return 0;
        }
        const auto* p = reinterpret_cast<const CandidatePair*>(pairs);
        st->out->assign(p, p + n);
        return 0;
    } catch (...) {
        st->err = std::current_exception();
        return 1;
    }
}

} // namespace

CCDKIT_EXPORT CcdReport ccd(const SceneStep& scene, const PipelineConfig& cfg)
{
    cfg.validate();
    // SceneStep::validate's element checks run on the device right after the
    // upload (k_validate_scene, same first-failure order and messages); only
    // the snapshot-length check needs the host containers
    if (scene.vertices_t0.size() != scene.vertices_t1.size())
        throw InvalidInput("vertex snapshots differ in length");
    const ccdk_pipeline_cfg c = to_c(cfg);
    ccdk_report r {};
    std::vector<CandidatePair> cands;
    CandidateSink sink { &cands, nullptr };
    SequenceGuard g(sequence_mutex());
    const int rc = ccdk_ccd_into(context(), vdata(scene.vertices_t0), vdata(scene.vertices_t1),
                                 scene.vertices_t0.size(), edata(scene), scene.edges.size(), fdata(scene),
                                 scene.faces.size(), &c, &r, candidate_sink, &sink);
    if (sink.err)
        std::rethrow_exception(sink.err);
    check(rc);
    CcdReport rep = to_report(r, false);
    rep.candidates = std::move(cands);
    return rep;
}

CCDKIT_EXPORT ToiResult run_batched(const SceneStep& scene, const std::vector<Aabb>& boxes,
                                    const PipelineConfig& cfg, BatchTrace& trace, CcdReport* report)
{
    cfg.validate();
    if (scene.vertices_t0.size() != scene.vertices_t1.size()) // element checks: on the device
        throw InvalidInput("vertex snapshots differ in length");
    // the caller's boxes, any order, through the device broad phase
    // (ccdk_run_batched: batches halve sorted positions, raw ones for bf)
    const BoxArrays b(boxes);
    const ccdk_pipeline_cfg c = to_c(cfg);
    ccdk_report r {};
    std::vector<CandidatePair> cands;
    CandidateSink sink { &cands, nullptr };
    SequenceGuard g(sequence_mutex());
    const int rc = ccdk_run_batched(context(), vdata(scene.vertices_t0), vdata(scene.vertices_t1),
                                    scene.vertices_t0.size(), edata(scene), scene.edges.size(), fdata(scene),
                                    scene.faces.size(), b.mn.data(), b.mx.data(), b.kind.data(), b.index.data(),
                                    boxes.size(), &c, &r, report ? candidate_sink : nullptr, &sink);
    if (sink.err)
        std::rethrow_exception(sink.err);
    check(rc);
    trace.broad_batches += r.broad_batches;
    trace.narrow_batches += r.batch_count;
    if (report) { // exactly the fields the reference's run_batched writes (pipeline.cpp:198-214)
        const CcdReport fresh = to_report(r, false);
        report->toi = fresh.toi;
        report->candidate_count = fresh.candidate_count;
        report->query_count = fresh.query_count;
        report->batch_count = std::max<std::size_t>(1, trace.narrow_batches);
        report->per_stage_times["BP"] = r.t_bp;
        report->per_stage_times["SO/CD"] = r.t_socd;
        report->per_stage_times["NP"] = r.t_np;
        report->tracked_peak_bytes = std::max(report->tracked_peak_bytes, fresh.tracked_peak_bytes);
        report->candidates = std::move(cands);
        report->real_record_sizes = fresh.real_record_sizes;
    }
    return { r.toi, r.tolerance_hit != 0, r.zero_toi_diagnostic != 0 };
}

CCDKIT_EXPORT CcdReport ccd_no_zero_toi(const SceneStep& scene, const PipelineConfig& cfg)
{
    if (!cfg.narrow.no_zero_toi)
        throw ConfigError("ccd_no_zero_toi: cfg.narrow.no_zero_toi must be set");
    if (scene.vertices_t0.size() != scene.vertices_t1.size()) // element checks: on the device
        throw InvalidInput("vertex snapshots differ in length");
    const ccdk_pipeline_cfg c = to_c(cfg);
    ccdk_report r {};
    SequenceGuard g(sequence_mutex());
    check(ccdk_ccd_no_zero_toi(context(), vdata(scene.vertices_t0), vdata(scene.vertices_t1),
                               scene.vertices_t0.size(), edata(scene), scene.edges.size(), fdata(scene),
                               scene.faces.size(), &c, &r));
    return to_report(r, true);
}

CCDKIT_EXPORT std::vector<double> query_min_separations(const std::vector<NarrowQuery>& queries,
                                                        const PipelineConfig& cfg)
{
    const size_t n = queries.size();
    std::vector<double> out(n);
    if (!n)
        return out;
    std::vector<uint8_t> kind(n);
    std::vector<double> pts(24 * n);
    for (size_t i = 0; i < n; ++i)
        flatten(queries[i], kind[i], &pts[24 * i]);
    const ccdk_pipeline_cfg c = to_c(cfg);
    check(ccdk_query_min_separations(context(), kind.data(), pts.data(), n, &c, out.data()));
    return out;
}

// --------------------------------------------------------------- distance

static double distance_one(uint8_t kind, const Vec3& a, const Vec3& b, const Vec3& c, const Vec3& d)
{
    double pts[24] = {};
    const Vec3* v[4] = { &a, &b, &c, &d };
    for (int i = 0; i < 4; ++i)
        for (int k = 0; k < 3; ++k)
            pts[3 * i + k] = (*v[i])[k];
    ccdk_pipeline_cfg cfg = to_c(PipelineConfig {});
    cfg.min_sep_mode = CCDK_MINSEP_RELATIVE;
    cfg.min_sep_fraction = 1.0;
    double out = 0;
    check(ccdk_query_min_separations(context(), &kind, pts, 1, &cfg, &out));
    return out;
}

CCDKIT_EXPORT double point_triangle_distance(const Vec3& p, const Vec3& a, const Vec3& b, const Vec3& c)
{
    return distance_one(CCDK_QUERY_VF, p, a, b, c);
}

CCDKIT_EXPORT double segment_segment_distance(const Vec3& p0, const Vec3& p1, const Vec3& q0, const Vec3& q1)
{
    return distance_one(CCDK_QUERY_EE, p0, p1, q0, q1);
}

} // namespace ccdkit
