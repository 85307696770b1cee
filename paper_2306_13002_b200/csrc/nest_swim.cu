// Registration of the swim nest functions (generated bodies: gen/swim.cuh).
#include "registry.hpp"
#include "kernels/march.cuh"
#include "kernels/stream.cuh"
#include "gen/swim.cuh"

namespace acs {

void register_swim() {
    {
        static Entry e;
        e.kernel_id = "swim.c:calc1:0";
        e.function = "calc1";
        describe<gen::calc1>(e, "swim.c", 0);
        fill_naive<gen::calc1, double>(e, 0);
        fill_naive_multi<gen::calc1, double, 2>(e, 0);
        fill_naive_multi<gen::calc1, double, 4>(e, 0);
        fill_march<gen::calc1, double, 0, 128, 1, 128, 1, 3>(e, 0);
        fill_march<gen::calc1, double, 0, 128, 1, 64, 1, 3>(e, 0);
        fill_march<gen::calc1, double, 0, 64, 1, 64, 1, 4>(e, 0);
        fill_march<gen::calc1, double, 0, 128, 1, 128, 1, 3, 1, 4>(e, 0);   // 4-row chunks (kchunk sweep)
        register_entry(&e);
    }
    {
        static Entry e;
        e.kernel_id = "swim.c:calc2:1";
        e.function = "calc2";
        describe<gen::calc2>(e, "swim.c", 1);
        fill_naive<gen::calc2, double>(e, 0);
        fill_march<gen::calc2, double, 0, 128, 1, 128, 1, 3>(e, 0);
        fill_march<gen::calc2, double, 0, 128, 1, 64, 1, 3>(e, 0);
        fill_march<gen::calc2, double, 0, 64, 1, 64, 1, 4>(e, 0);
        fill_march<gen::calc2, double, 0, 128, 1, 128, 1, 5>(e, 0);
        fill_march<gen::calc2, double, 0, 128, 1, 128, 1, 7>(e, 0);
        fill_march<gen::calc2, double, 0, 128, 1, 64, 1, 3, 2>(e, 0);
        register_entry(&e);
    }
    {
        static Entry e;
        e.kernel_id = "swim.c:calc3:2";
        e.function = "calc3";
        describe<gen::calc3>(e, "swim.c", 2);
        fill_naive<gen::calc3, double>(e, 0);
        fill_naive_multi<gen::calc3, double, 2>(e, 0);
        fill_naive_multi<gen::calc3, double, 4>(e, 0);
        fill_stream<gen::calc3, double, 128, 3>(e, 0);
        fill_stream<gen::calc3, double, 256, 4>(e, 0);
        fill_march<gen::calc3, double, 0, 128, 1, 128, 1, 3>(e, 0);
        fill_march<gen::calc3, double, 0, 128, 1, 64, 1, 3>(e, 0);
        fill_march<gen::calc3, double, 0, 64, 1, 64, 1, 4>(e, 0);
        register_entry(&e);
    }
}

}  // namespace acs
