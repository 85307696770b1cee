// Registration of the d3q19 nest functions (generated bodies: gen/d3q19.cuh).
#include "registry.hpp"
#include "kernels/march.cuh"
#include "kernels/stream.cuh"
#include "gen/d3q19.cuh"

namespace acs {

void register_d3q19() {
    {
        static Entry e;
        e.kernel_id = "d3q19.c:stream_collide:0";
        e.function = "stream_collide";
        describe<gen::stream_collide>(e, "d3q19.c", 0);
        fill_naive<gen::stream_collide, double>(e, 0);
        fill_naive_occ<gen::stream_collide, double, 3>(e, 0);
        fill_naive_occ<gen::stream_collide, double, 4>(e, 0);
        fill_stream<gen::stream_collide, double, 128, 3>(e, 0);
        fill_march<gen::stream_collide, double, 1, 64, 4, 64, 4, 1>(e, 0);
        fill_march<gen::stream_collide, double, 1, 64, 2, 64, 2, 3>(e, 0);
        fill_march<gen::stream_collide, double, 1, 32, 4, 32, 4, 3>(e, 0);
        e.soa_last_dim = true;
        register_entry(&e);
    }
}

}  // namespace acs
