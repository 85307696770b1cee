// Registration of the clover nest functions (generated bodies: gen/clover.cuh).
#include "registry.hpp"
#include "kernels/march.cuh"
#include "kernels/stream.cuh"
#include "gen/clover.cuh"

namespace acs {

void register_clover() {
    {
        static Entry e;
        e.kernel_id = "clover.c:ideal_gas:0";
        e.function = "ideal_gas";
        describe<gen::ideal_gas>(e, "clover.c", 0);
        e.row_offset = true;   // sector-aligned rows (x starts at 2: a 16-byte shift)
        fill_naive<gen::ideal_gas, double>(e, 0);
        fill_naive_multi<gen::ideal_gas, double, 2>(e, 0);
        fill_naive_multi<gen::ideal_gas, double, 4>(e, 0);
        fill_stream<gen::ideal_gas, double, 128, 3>(e, 0);
        fill_stream<gen::ideal_gas, double, 256, 4>(e, 0);
        fill_march<gen::ideal_gas, double, 0, 128, 1, 128, 1, 3>(e, 0);
        fill_march<gen::ideal_gas, double, 0, 128, 1, 64, 1, 3>(e, 0);
        fill_march<gen::ideal_gas, double, 0, 64, 1, 64, 1, 4>(e, 0);
        register_entry(&e);
    }
    {
        static Entry e;
        e.kernel_id = "clover.c:pdv_predict:1";
        e.function = "pdv_predict";
        describe<gen::pdv_predict>(e, "clover.c", 1);
        fill_naive<gen::pdv_predict, double>(e, 0);
        fill_march<gen::pdv_predict, double, 0, 128, 1, 128, 1, 3>(e, 0);
        fill_march<gen::pdv_predict, double, 0, 128, 1, 64, 1, 3>(e, 0);
        fill_march<gen::pdv_predict, double, 0, 64, 1, 64, 1, 4>(e, 0);
        fill_march<gen::pdv_predict, double, 0, 128, 1, 128, 1, 5>(e, 0);
        fill_march<gen::pdv_predict, double, 0, 128, 1, 128, 1, 7>(e, 0);
        fill_march<gen::pdv_predict, double, 0, 128, 1, 128, 1, 3, 1, 12>(e, 0);   // 12-row chunks
        register_entry(&e);
    }
    {
        static Entry e;
        e.kernel_id = "clover.c:advec_cell_x:2";
        e.function = "advec_cell_x";
        describe<gen::advec_cell_x>(e, "clover.c", 2);
        fill_naive<gen::advec_cell_x, double>(e, 0);
        fill_march<gen::advec_cell_x, double, 0, 128, 1, 128, 1, 3>(e, 0);
        fill_march<gen::advec_cell_x, double, 0, 128, 1, 64, 1, 3>(e, 0);
        fill_march<gen::advec_cell_x, double, 0, 64, 1, 64, 1, 4>(e, 0);
        fill_march<gen::advec_cell_x, double, 0, 128, 1, 128, 1, 5>(e, 0);
        fill_march<gen::advec_cell_x, double, 0, 128, 1, 128, 1, 7>(e, 0);
        fill_march<gen::advec_cell_x, double, 0, 128, 1, 128, 1, 3, 1, 12>(e, 0);   // 12-row chunks
        register_entry(&e);
    }
}

}  // namespace acs
