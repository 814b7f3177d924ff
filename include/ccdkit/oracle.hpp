// ccdkit drop-in (B200 build): declarations of the reference's exact
// ground-truth oracle (proj/include/ccdkit/oracle.hpp).  The oracle is NOT
// part of the B200 build — it is exact rational arithmetic (GMP), test and
// audit infrastructure, not the CCD path.  Its implementation is the
// reference's own proj/src/oracle.cpp, linked by whoever wants ground truth
// (the audit tool ccdbench, the reference's tests).  bench_scene() in
// libccdkit.so binds ground_truth_pairs() weakly: without an oracle linked,
// RunSpec::oracle_enabled throws ConfigError.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ccdkit/broadphase.hpp"

namespace ccdkit {

struct OracleVerdict {
    bool colliding = false;
    bool indeterminate = false;
    double root_lo = 0.0; // exact earliest valid root, rounded down (when colliding)
    double root_hi = 0.0; // ... rounded up
    bool root_exact = false;
    double root_width = 0.0;
    double margin = 0.0; // certified lower bound on min ||F||_inf (not colliding)
    bool margin_valid = false;
    std::string root_lo_dec;
    std::string root_hi_dec;
};

struct OracleOptions {
    unsigned precision_bits = 128;
    unsigned max_refine_bits = 640;
    bool compute_margin = true;
    unsigned margin_iterations = 200;
    double margin_target = 1e-3;
};

OracleVerdict oracle_toi(const NarrowQuery& query, const OracleOptions& opts = {});

inline OracleVerdict oracle_toi(const NarrowQuery& query, unsigned precision_bits)
{
    OracleOptions opts;
    opts.precision_bits = precision_bits;
    return oracle_toi(query, opts);
}

struct GroundTruthPair {
    CandidatePair pair;
    OracleVerdict verdict;
};

struct GroundTruth {
    std::vector<GroundTruthPair> colliding;   // sorted by pair
    std::vector<CandidatePair> indeterminate; // excluded from FN accounting
    std::size_t pairs_evaluated = 0;
    std::size_t pairs_prefiltered = 0;
};

GroundTruth ground_truth_pairs(const SceneStep& scene, const OracleOptions& opts = {},
                               unsigned threads = 1);

std::uint64_t query_hash(const NarrowQuery& query);

std::string verdict_to_json(const NarrowQuery& query, const OracleVerdict& verdict);

} // namespace ccdkit
