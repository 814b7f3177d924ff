// Breakdown of the drop-in's end-to-end ccd() time on the GPU box (scratch
// measurement tool): pageable upload, step without candidates, step with a
// no-op candidate sink, step with the report's vector fill, and the host-only
// cost of filling a std::vector<CandidatePair> of the same size.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "ccdk.h"
#include "ccdkit/bench.hpp"

using Clock = std::chrono::steady_clock;
static double ms(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

static int noop_sink(void*, const uint64_t*, uint64_t) { return 0; }
static int fill_sink(void* u, const uint64_t* p, uint64_t n)
{
    if (!p)
        return 0;
    auto* v = static_cast<std::vector<ccdkit::CandidatePair>*>(u);
    const auto* c = reinterpret_cast<const ccdkit::CandidatePair*>(p);
    v->assign(c, c + n);
    return 0;
}

int main()
{
    const ccdkit::SceneStep s = ccdkit::make_cloth_scene(410, 410, 0.02, 1.0, 4);
    ccdk_ctx* ctx = nullptr;
    ccdk_ctx_create(0, &ctx);
    ccdk_pipeline_cfg cfg {};
    cfg.narrow.delta = 1e-6; cfg.narrow.t_max = 1.0; cfg.narrow.max_splits = 1ull << 20;
    cfg.memory_budget = ~0ull / 4; cfg.rs_params = 56; cfg.rs_query = 192; cfg.rs_interval = 252; cfg.rs_pair_ints = 8;
    cfg.min_sep_fraction = 0.2; cfg.threads = 1; cfg.inflation = 0.01;
    const double* v0 = s.vertices_t0[0].data(); const double* v1 = s.vertices_t1[0].data();
    const uint32_t* e = s.edges[0].data(); const uint32_t* f = s.faces[0].data();
    const uint64_t nv = s.vertices_t0.size(), ne = s.edges.size(), nf = s.faces.size();
    ccdk_report r {};
    void* dbuf; cudaMalloc(&dbuf, 64 << 20);
    for (int rep = 0; rep < 4; ++rep) {
        auto a = Clock::now();
        cudaMemcpy(dbuf, v0, nv * 24, cudaMemcpyHostToDevice);
        cudaMemcpy(dbuf, v1, nv * 24, cudaMemcpyHostToDevice);
        cudaMemcpy(dbuf, e, ne * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dbuf, f, nf * 12, cudaMemcpyHostToDevice);
        auto b = Clock::now();
        ccdk_ccd(ctx, v0, v1, nv, e, ne, f, nf, &cfg, &r);
        auto c = Clock::now();
        ccdk_ccd_into(ctx, v0, v1, nv, e, ne, f, nf, &cfg, &r, noop_sink, nullptr);
        auto d = Clock::now();
        std::vector<ccdkit::CandidatePair> out;
        ccdk_ccd_into(ctx, v0, v1, nv, e, ne, f, nf, &cfg, &r, fill_sink, &out);
        auto g = Clock::now();
        std::vector<uint64_t> src(2 * r.candidate_count, 1);
        auto h = Clock::now();
        std::vector<ccdkit::CandidatePair> host;
        fill_sink(&host, src.data(), r.candidate_count);
        auto i = Clock::now();
        const ccdkit::CcdReport full = ccdkit::ccd(s, [] { ccdkit::PipelineConfig p; p.inflation = 0.01; return p; }());
        auto j = Clock::now();
        ccdk_scene_upload(ctx, v0, v1, nv, e, ne, f, nf);
        auto k2 = Clock::now();
        ccdk_report rr {};
        ccdk_ccd_resident(ctx, &cfg, 0, 1, &rr);
        auto l2 = Clock::now();
        std::printf("  resident: upload %.2f ms, step %.2f ms (device %.2f)\n", ms(j, k2), ms(k2, l2), rr.ms_total);
        std::printf("pageable H2D %.2f | ccdk_ccd %.2f (device total %.2f) | into+noop %.2f | into+fill %.2f | host fill %.2f | ccdkit::ccd %.2f ms (n=%llu)\n",
                    ms(a, b), ms(b, c), r.ms_total, ms(c, d), ms(d, g), ms(h, i), ms(i, j), (unsigned long long)r.candidate_count);
    }
    return 0;
}
