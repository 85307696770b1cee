// Registration of the wave4 nest functions (generated bodies: gen/wave4.cuh).
#include "registry.hpp"
#include "kernels/march.cuh"
#include "kernels/tbwave.cuh"
#include "gen/wave4.cuh"

namespace acs {

void register_wave4() {
    {
        static Entry e;
        e.kernel_id = "wave4.c:wave4:0";
        e.function = "wave4";
        describe<gen::wave4>(e, "wave4.c", 0);
        e.row_offset = true;   // sector-aligned rows (TMA x-origin shift, aligned origin follows it)
        fill_naive<gen::wave4, double>(e, 0);
        fill_march<gen::wave4, double, 0, 32, 8, 32, 8, 3>(e, 0);
        fill_march<gen::wave4, double, 0, 32, 16, 32, 4, 3>(e, 0);
        fill_naive<gen::wave4_f32, float>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 64, 8, 64, 8, 3>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 64, 8, 64, 2, 3>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 64, 16, 64, 4, 2>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 128, 8, 32, 8, 2, 4>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 64, 8, 64, 2, 4>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 64, 16, 16, 16, 2, 4>(e, 1);
        fill_march<gen::wave4_f32, float, 0, 32, 16, 32, 4, 3>(e, 1);
        // two leapfrog steps per launch (kernels/tbwave.cuh, acs_launch_leapfrog2), fp32 config
        fill_tbw<gen::wave4_f32, float, gen::wave4_f32::ARR_u, gen::wave4_f32::ARR_up, gen::wave4_f32::ARR_un,
                 gen::wave4_f32::ARR_vel2, 32, 16, 2, 3>(e, 1);
        register_entry(&e);
    }
}

}  // namespace acs
