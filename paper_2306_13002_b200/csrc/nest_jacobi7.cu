// Registration of the jacobi7 nest functions (generated bodies: gen/jacobi7.cuh).
#include "registry.hpp"
#include "kernels/march.cuh"
#include "kernels/tblock.cuh"
#include "gen/jacobi7.cuh"

namespace acs {

void register_jacobi7() {
    {
        static Entry e;
        e.kernel_id = "jacobi7.c:jacobi7:0";
        e.function = "jacobi7";
        describe<gen::jacobi7>(e, "jacobi7.c", 0);
        e.row_offset = true;   // sector-aligned rows; the TMA maps start adj elements earlier
        fill_naive<gen::jacobi7, double>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 8, 128, 2, 2>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 8, 128, 2, 3>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 8, 128, 4, 3>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 4, 128, 2, 2>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 16, 128, 4, 2>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 4, 128, 2, 3>(e, 0);
        fill_march<gen::jacobi7, double, 0, 128, 16, 64, 4, 2, 2>(e, 0);
        // two sweeps per launch (kernels/tblock.cuh): the default, then ACS_TB_CFG=1..5 alternatives (5: x neighbours by warp shuffle)
        fill_tb2<gen::jacobi7, double, TbCfg<32, 16, 2, 4, 4>, TbCfg<32, 16, 1, 4, 3>, TbCfg<32, 32, 2, 4, 2>,
                 TbCfg<64, 16, 2, 4, 2>, TbCfg<32, 16, 4, 4, 4>, TbCfg<32, 16, 2, 4, 4, 1>>(e, 0);
        register_entry(&e);
    }
}

}  // namespace acs
