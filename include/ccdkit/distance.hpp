// ccdkit drop-in (B200 build): t = 0 primitive distances
// (proj/include/ccdkit/distance.hpp), evaluated by the device kernel behind
// ccdk_query_min_separations.
#pragma once

#include "ccdkit/core.hpp"

namespace ccdkit {

double point_triangle_distance(const Vec3& p, const Vec3& a, const Vec3& b, const Vec3& c);
double segment_segment_distance(const Vec3& p0, const Vec3& p1, const Vec3& q0, const Vec3& q1);

} // namespace ccdkit
