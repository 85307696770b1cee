// zsolve sliced configuration (128 x 2, k-chunk 32, unroll 2), own translation unit.
#include "registry.hpp"
#include "kernels/sliced.cuh"
#include "gen/zsolve.cuh"

namespace acs {

void fill_zsolve_sliced_b(Entry& e) { fill_sliced<gen::z_solve_lhs, double, 128, 2, 32, 2>(e, 0); }

}  // namespace acs
