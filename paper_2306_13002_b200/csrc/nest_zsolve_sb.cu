// zsolve sliced configuration (64 x 4, k-chunk 16), own translation unit.
#include "registry.hpp"
#include "kernels/sliced.cuh"
#include "gen/zsolve.cuh"

namespace acs {

void fill_zsolve_sliced_b(Entry& e) { fill_sliced<gen::z_solve_lhs, double, 64, 4, 16>(e, 0); }

}  // namespace acs
