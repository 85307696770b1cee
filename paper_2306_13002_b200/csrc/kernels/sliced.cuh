// sliced.cuh — the component-sliced skeleton ("sliced" schedule).
//
// For nests whose stores fall into independent component groups (the
// lowering's slice analysis: zsolve's 25 5x5-block entries, each reading
// only its own fjacZ[m][n] / njacZ[m][n] fields), a thread owns ONE slice at
// one (i, j) column and marches the outermost loop over a chunk of planes:
//
//   * 25x the threads of the point-per-thread skeleton at 1/25 of the live
//     state each — a handful of registers, full occupancy, and every SM has
//     thousands of independent loads in flight;
//   * the k-1 / k / k+1 re-reads of a component field hit the thread's own
//     recent lines in L1 (ld.global.nc), so each element crosses HBM once.
//
// Slices of one form are emitted by the lowering in the form's statement
// order; a CTA runs one slice, so the slice switch is uniform per CTA.
#pragma once

#include "../acs_device.cuh"
#include "../registry.hpp"

namespace acs {

// the k march of one slice, the slice a compile-time constant: no switch in
// the loop, so the loads of several planes can be issued ahead (unroll)
template <class NS, class T, int FORM, int S>
__device__ __forceinline__ void march_slice(NaiveMem<NS, T, FORM == ACS_ORIGINAL>& m, const KernelArgs<NS>& args,
                                            int* pt, int slice, int kb, int ke) {
    if constexpr (S < NS::nslices[FORM]) {
        if (slice == S) {
#pragma unroll 4
            for (int k = kb; k < ke; ++k) {
                pt[0] = k;
                NS::template body_slice<FORM, S>(m, args.s, pt);
            }
        } else {
            march_slice<NS, T, FORM, S + 1>(m, args, pt, slice, kb, ke);
        }
    }
}

template <class NS, class T, int FORM, int BX, int BY>
__global__ void __launch_bounds__(BX* BY) sliced_kernel(const __grid_constant__ KernelArgs<NS> args, int kchunk) {
    static_assert(NS::NLOOP == 3, "sliced skeleton: 3-D nests");
    constexpr int NSL = NS::nslices[FORM];
    const int slice = (int)(blockIdx.z % NSL);
    const int chunk = (int)(blockIdx.z / NSL);
    const int x = args.lo[2] + (int)(blockIdx.x * BX + threadIdx.x);
    const int y = args.lo[1] + (int)(blockIdx.y * BY + threadIdx.y);
    if (x >= args.hi[2] || y >= args.hi[1]) return;
    const int kb = args.lo[0] + chunk * kchunk;
    const int ke = min(kb + kchunk, (int)args.hi[0]);
    int pt[3];
    pt[1] = y;
    pt[2] = x;
    NaiveMem<NS, T, FORM == ACS_ORIGINAL> m{args, pt};
    march_slice<NS, T, FORM, 0>(m, args, pt, slice, kb, ke);
}

template <class NS, class T, int FORM, int BX, int BY, int KCH>
acs_status launch_sliced(const LaunchReq& r) {
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    constexpr int NSL = NS::nslices[FORM];
    const long long nx = ka.hi[2] - ka.lo[2], ny = ka.hi[1] - ka.lo[1], nz = ka.hi[0] - ka.lo[0];
    const long long chunks = (nz + KCH - 1) / KCH;
    dim3 grid((unsigned)((nx + BX - 1) / BX), (unsigned)((ny + BY - 1) / BY), (unsigned)(chunks * NSL));
    sliced_kernel<NS, T, FORM, BX, BY><<<grid, dim3(BX, BY, 1), 0, r.stream>>>(ka, KCH);
    return check_launch("sliced");
}

template <class NS, class T, int BX, int BY, int KCH>
void fill_sliced(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_sliced<NS, T, 0, BX, BY, KCH>;
    e.launch[prec][1][slot] = &launch_sliced<NS, T, 1, BX, BY, KCH>;
    e.launch[prec][2][slot] = &launch_sliced<NS, T, 2, BX, BY, KCH>;
    e.launch[prec][3][slot] = &launch_sliced<NS, T, 3, BX, BY, KCH>;
    e.launch[prec][4][slot] = &launch_sliced<NS, T, 4, BX, BY, KCH>;
    e.sched_name[prec][slot] = "sliced " + std::to_string(NS::nslices[4]) + " components, block " +
                               std::to_string(BX) + "x" + std::to_string(BY) + ", k-chunk " + std::to_string(KCH);
    for (int v = 0; v < 5; ++v)
        if (e.best[prec][v] == 0 && v != ACS_ORIGINAL) e.best[prec][v] = slot;
}

}  // namespace acs
