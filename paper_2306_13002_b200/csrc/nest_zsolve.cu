// Registration of the zsolve nest function (generated body: gen/zsolve.cuh).
// NPB-BT z_solve LHS: 50 loaded component fields (fjacZ/njacZ at k-1, k, k+1)
// and 75 stored ones per point; every (m, n[, side]) component is its own
// contiguous 3-D field, so the naive skeleton's loads are already coalesced
// along j and the k-neighbour re-reads are L2 hits (three planes of the 50
// loaded fields = 80 MB at 258^2 < 126 MB L2); the march skeleton stages the
// 25-component boxes of both jacobians per k-plane through TMA; the sliced
// skeleton gives each of the 25 independent (m, n) components its own
// threads, marching k with the re-reads served by L1.
//
// The sliced configurations are instantiated in their own translation units
// (nest_zsolve_s*.cu) so nvcc compiles them in parallel.
#include "registry.hpp"
#include "gen/zsolve.cuh"

namespace acs {

void fill_zsolve_sliced_a(Entry& e);
void fill_zsolve_sliced_b(Entry& e);
void fill_zsolve_sliced_c(Entry& e);

void register_zsolve() {
    static Entry e;
    e.kernel_id = "zsolve.c:z_solve_lhs:0";
    e.function = "z_solve_lhs";
    describe<gen::z_solve_lhs>(e, "zsolve.c", 0);
    e.row_offset = true;   // naive / sliced skeletons only: sector-aligned interior rows
    fill_naive<gen::z_solve_lhs, double>(e, 0);
    fill_zsolve_sliced_a(e);
    fill_zsolve_sliced_b(e);
    fill_zsolve_sliced_c(e);
    register_entry(&e);
}

}  // namespace acs
