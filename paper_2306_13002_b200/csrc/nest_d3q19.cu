// Registration of the d3q19 nest functions (generated bodies: gen/d3q19.cuh).
#include "registry.hpp"
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
        // no march slots: the TMA cannot describe the sector-aligned q-major
        // layout (24-byte start offset), and round 1's march slots only ever
        // ran the naive fallback
        e.soa_last_dim = true;
        register_entry(&e);
    }
}

}  // namespace acs
