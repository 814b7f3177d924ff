// ccdkit drop-in (B200 build): swept boxes (proj/include/ccdkit/aabb.hpp).
// build_boxes runs the K1 kernel through ccdk_build_boxes (include/ccdk.h).
#pragma once

#include <array>
#include <vector>

#include "ccdkit/scene.hpp"

namespace ccdkit {

// Largest float r with (double)r <= x / smallest float r with (double)r >= x.
float round_down_reduced(double x);
float round_up_reduced(double x);

struct Aabb {
    std::array<float, 3> min_corner {};
    std::array<float, 3> max_corner {};
    PrimitiveId owner;

    bool overlaps_axis(const Aabb& o, int axis) const
    {
        return min_corner[axis] <= o.max_corner[axis] && o.min_corner[axis] <= max_corner[axis];
    }
    bool overlaps(const Aabb& o) const
    {
        return overlaps_axis(o, 0) && overlaps_axis(o, 1) && overlaps_axis(o, 2);
    }
};

// Floor for the padding of a zero-extent axis when inflation > 0.
inline constexpr double kZeroExtentInflation = 1e-12;

// One box per vertex, edge, face (that order, each by index); fp64 extents
// over both snapshots, per-axis inflation, outward rounding to fp32.
// `threads` is accepted for signature compatibility and ignored.
std::vector<Aabb> build_boxes(const SceneStep& scene, double inflation = 0.0, unsigned threads = 1);

} // namespace ccdkit
