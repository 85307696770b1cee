// zsolve sliced configuration (128 x 1, k-chunk 64, unroll 2), own translation unit.
#include "registry.hpp"
#include "kernels/sliced.cuh"
#include "gen/zsolve.cuh"

namespace acs {

void fill_zsolve_sliced_c(Entry& e) { fill_sliced<gen::z_solve_lhs, double, 128, 1, 64, 2>(e, 0); }

}  // namespace acs
