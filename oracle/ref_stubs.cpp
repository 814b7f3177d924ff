// TEST INFRASTRUCTURE ONLY.  The reference's exact oracle (oracle.cpp) needs
// Boost.Multiprecision + GMP headers that are absent here, so
// the one oracle symbol bench.cpp links against is stubbed; the generators in
// bench.cpp (make_cloth_scene / make_box_soup) are what oracle/_ref uses.
#include <stdexcept>

#include "ccdkit/oracle.hpp"

namespace ccdkit_ref {
GroundTruth ground_truth_pairs(const SceneStep&, const OracleOptions&, unsigned)
{
    throw std::runtime_error("oracle.cpp is not buildable here (no Boost/GMP headers)");
}
} // namespace ccdkit_ref
