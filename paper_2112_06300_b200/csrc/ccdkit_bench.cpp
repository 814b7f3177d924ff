// End-to-end timing harness for the drop-in: the reference's own entry point
// ccdkit::ccd(const SceneStep&, const PipelineConfig&) (proj/src/
// pipeline.cpp:218-232) called through libccdkit.so exactly as a user of the
// reference would call it — SceneStep in ordinary (pageable) host vectors,
// CcdReport returned by value with every CandidatePair (pipeline.cpp:209).
// bench.py drives it through this small C entry so the timed region is the
// C++ call alone (scene construction happens once, outside).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

#include "ccdkit/pipeline.hpp"

#define BENCH_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

struct Bench {
    ccdkit::SceneStep scene;
    ccdkit::PipelineConfig cfg;
};

} // namespace

BENCH_EXPORT const char* ccdkit_bench_last_error() { return g_err.c_str(); }

BENCH_EXPORT void* ccdkit_bench_prepare(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                                        uint64_t ne, const uint32_t* f, uint64_t nf, double inflation)
{
    auto b = std::make_unique<Bench>();
    b->scene.vertices_t0.resize(nv);
    b->scene.vertices_t1.resize(nv);
    b->scene.edges.resize(ne);
    b->scene.faces.resize(nf);
    if (nv) {
        std::memcpy(b->scene.vertices_t0.data(), v0, nv * 24);
        std::memcpy(b->scene.vertices_t1.data(), v1, nv * 24);
    }
    if (ne)
        std::memcpy(b->scene.edges.data(), e, ne * 8);
    if (nf)
        std::memcpy(b->scene.faces.data(), f, nf * 12);
    b->cfg.inflation = inflation;
    return b.release();
}

BENCH_EXPORT void ccdkit_bench_free(void* h) { delete static_cast<Bench*>(h); }

// One ccdkit::ccd call: wall time (ms) of the synchronous call, candidate
// count, the report's ToI, and an order-sensitive checksum of the returned
// candidate list (so the caller can compare it with the device-resident run).
BENCH_EXPORT int ccdkit_bench_run(void* h, double* ms, uint64_t* candidates, double* toi, uint64_t* checksum)
{
    try {
        Bench& b = *static_cast<Bench*>(h);
        const auto t0 = std::chrono::steady_clock::now();
        const ccdkit::CcdReport rep = ccdkit::ccd(b.scene, b.cfg);
        const auto t1 = std::chrono::steady_clock::now();
        *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *candidates = rep.candidates.size();
        *toi = rep.toi.toi;
        uint64_t x = 1469598103934665603ull;
        for (const auto& c : rep.candidates) {
            const uint64_t l = (uint64_t(c.left.kind) << 32) | c.left.index;
            const uint64_t r = (uint64_t(c.right.kind) << 32) | c.right.index;
            x = (x ^ l) * 1099511628211ull;
            x = (x ^ r) * 1099511628211ull;
        }
        *checksum = x;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
