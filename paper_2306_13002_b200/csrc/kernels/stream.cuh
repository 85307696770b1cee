// stream.cuh — the per-thread asynchronous-prefetch skeleton ("stream" schedule).
//
// For nests whose loads are POINT-LOCAL — every loaded element sits at the
// point's own loop coordinates, possibly at several component subscripts
// (the 19 D3Q19 distributions of a cell, swim calc3's in-place time filter,
// ideal_gas) — there is no reuse to tile; what limits HBM throughput is how
// many bytes are in flight per SM.  Register-held loads cap that at the
// occupancy the body's register footprint allows (96 regs for D3Q19 = 16
// warps/SM).  Here each thread instead prefetches the NEXT point's elements
// with cp.async (LDGSTS) into its own shared-memory slots, S-1 points ahead,
// while it computes the current one from shared memory.  A thread only ever
// reads slots it filled itself, so no barrier is needed: cp.async.wait_group
// makes a thread's own copies visible to it.
//
// Thread mapping: a CTA of BX threads covers BX consecutive points of the
// innermost loop and walks a chunk of rows (the outer loops, flattened).
#pragma once

#include "../acs_device.cuh"
#include "../registry.hpp"

namespace acs {

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <class NS>
struct StreamPlan {
    static constexpr int NL = NS::NLOOP;
    // point-local: loaded, never stored, all loop-variable subscripts at offset 0
    static constexpr bool local(int a) {
        if (!NS::stageable(a)) return false;
        for (int p = 0; p < NS::ndim(a); ++p) {
            const int s = NS::ld_sig(a, p);
            if (s >= 0 && (NS::ld_lo(a, p) != 0 || NS::ld_hi(a, p) != 0)) return false;
            if (s == -2) return false;
        }
        return true;
    }
    static constexpr int ncomp(int a) {
        int n = 1;
        for (int p = 0; p < NS::ndim(a); ++p)
            if (NS::ld_sig(a, p) == -1) n *= NS::ld_hi(a, p) - NS::ld_lo(a, p) + 1;
        return n;
    }
    static constexpr int slot0(int a) {
        int s = 0;
        for (int b = 0; b < a; ++b)
            if (local(b)) s += ncomp(b);
        return s;
    }
    static constexpr int nslot() { return slot0(NS::NARR); }
    static constexpr bool usable() {
        if (nslot() == 0) return false;
        for (int a = 0; a < NS::NARR; ++a)
            if (local(a)) {
                int nabs = 0;
                for (int p = 0; p < NS::ndim(a); ++p) nabs += NS::ld_sig(a, p) == -1;
                if (nabs > 1) return false;   // one component subscript at most
            }
        return true;
    }
};

template <class NS, class T, int BX, int S>
struct StreamMem {
    using P = StreamPlan<NS>;
    NaiveMem<NS, T, false> g;
    const double* stage;   // this thread's slots of the current stage: stage[slot * BX]

    template <int ARR>
    using elem_t = typename NaiveMem<NS, T, false>::template elem_t<ARR>;

    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const {
        if constexpr (P::local(ARR)) {
            constexpr int off[sizeof...(O)] = {O...};
            int comp = 0;
#pragma unroll
            for (int p = 0; p < (int)sizeof...(O); ++p)
                if (NS::ld_sig(ARR, p) == -1) comp = off[p] - NS::ld_lo(ARR, p);
            const double* slot = stage + (P::slot0(ARR) + comp) * BX;
            if constexpr (NS::is_int(ARR)) return *reinterpret_cast<const int*>(slot);
            else if constexpr (sizeof(T) == 4) return *reinterpret_cast<const float*>(slot);
            else return *slot;
        } else {
            return g.template ld<ARR, O...>();
        }
    }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... idx) const { return g.template ldx<ARR>(idx...); }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx_in(I... idx) const { return g.template ldx<ARR>(idx...); }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const { g.template st<ARR, O...>(v); }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const { g.template stx<ARR>(args...); }
};

// issue the cp.asyncs of every point-local element of point `pt` into `dst`
template <class NS, class T, int BX, int A>
__device__ __forceinline__ void stream_issue(const KernelArgs<NS>& args, const int* pt, double* dst) {
    using P = StreamPlan<NS>;
    if constexpr (A < NS::NARR) {
        if constexpr (P::local(A)) {
            long long base = 0;
            int cpos = -1;
#pragma unroll
            for (int p = 0; p < NS::ndim(A); ++p) {
                const int s = NS::ld_sig(A, p);
                if (s >= 0) base += (long long)pt[s] * args.arr[A].stride[p];
                else cpos = p;
            }
#pragma unroll
            for (int c = 0; c < P::ncomp(A); ++c) {
                const long long idx = base + (cpos >= 0 ? (long long)(NS::ld_lo(A, cpos) + c) * args.arr[A].stride[cpos] : 0);
                double* d = dst + (P::slot0(A) + c) * BX;
                if constexpr (NS::is_int(A)) cp_async4(d, reinterpret_cast<const int*>(args.arr[A].base) + idx);
                else if constexpr (sizeof(T) == 4) cp_async4(d, reinterpret_cast<const float*>(args.arr[A].base) + idx);
                else cp_async8(d, reinterpret_cast<const double*>(args.arr[A].base) + idx);
            }
        }
        stream_issue<NS, T, BX, A + 1>(args, pt, dst);
    }
}

template <class NS, class T, int FORM, int BX, int S>
__global__ void __launch_bounds__(BX) stream_kernel(const __grid_constant__ KernelArgs<NS> args, int rows_per_cta) {
    using P = StreamPlan<NS>;
    constexpr int NL = NS::NLOOP;
    extern __shared__ __align__(16) double sbuf[];   // [S][nslot][BX]
    const int tx = threadIdx.x;
    const int x = args.lo[NL - 1] + blockIdx.x * BX + tx;
    const bool xin = x < args.hi[NL - 1];
    // outer loops flattened to rows
    long long nrows = 1, ny = 1;
    if constexpr (NL >= 2) nrows = args.hi[0] - args.lo[0];
    if constexpr (NL == 3) {
        ny = args.hi[1] - args.lo[1];
        nrows *= ny;
    }
    const long long r0 = (long long)blockIdx.y * rows_per_cta;
    const long long r1 = r0 + rows_per_cta < nrows ? r0 + rows_per_cta : nrows;
    int pt[NL];
    pt[NL - 1] = x;
    auto set_row = [&](long long r) {
        if constexpr (NL == 3) {
            pt[0] = args.lo[0] + (int)(r / ny);
            pt[1] = args.lo[1] + (int)(r % ny);
        } else if constexpr (NL == 2) {
            pt[0] = args.lo[0] + (int)r;
        }
    };
    double* mine = sbuf + tx;
    constexpr int STAGE = P::nslot() * BX;
    // prologue: S-1 rows in flight
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        const long long r = r0 + s;
        if (xin && r < r1) {
            set_row(r);
            stream_issue<NS, T, BX, 0>(args, pt, mine + s * STAGE);
        }
        cp_async_commit();
    }
    int stage = 0;
    for (long long r = r0; r < r1; ++r) {
        const long long rn = r + S - 1;
        const int sn = (stage + S - 1) % S;
        if (xin && rn < r1) {
            set_row(rn);
            stream_issue<NS, T, BX, 0>(args, pt, mine + sn * STAGE);
        }
        cp_async_commit();
        cp_async_wait<S - 1>();   // this thread's copies for row r have landed
        if (xin) {
            set_row(r);
            StreamMem<NS, T, BX, S> m{NaiveMem<NS, T, false>{args, pt}, mine + stage * STAGE};
            NS::template body<FORM>(m, args.s, pt);
        }
        stage = stage + 1 == S ? 0 : stage + 1;
    }
    cp_async_wait<0>();
    if (args.sh.enabled) __threadfence_system();   // peer write-through visible before the step flag
}

template <class NS, class T, int FORM, int BX, int S>
acs_status launch_stream(const LaunchReq& r) {
    using P = StreamPlan<NS>;
    static_assert(P::usable(), "stream skeleton: no point-local loads");
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    constexpr int NL = NS::NLOOP;
    constexpr int smem = S * P::nslot() * BX * 8;
    auto kern = stream_kernel<NS, T, FORM, BX, S>;
    static std::atomic<unsigned long long> attr_done{0};
    set_smem_attr_once(kern, smem, attr_done);
    const long long nx = ka.hi[NL - 1] - ka.lo[NL - 1];
    long long nrows = 1;
    if (NL >= 2) nrows = ka.hi[0] - ka.lo[0];
    if (NL == 3) nrows *= ka.hi[1] - ka.lo[1];
    const long long xt = (nx + BX - 1) / BX;
    // ~16 CTAs per SM in total; each walks a chunk of rows
    long long want = (148LL * 16 + xt - 1) / xt;
    long long rpc = (nrows + want - 1) / want;
    if (rpc < 4) rpc = 4;
    if (rpc > nrows) rpc = nrows;
    dim3 grid((unsigned)xt, (unsigned)((nrows + rpc - 1) / rpc), 1);
    if (r.preload) return preload_fn((const void*)kern);
    kern<<<grid, BX, smem, r.stream>>>(ka, (int)rpc);
    return check_launch("stream");
}

template <class NS, class T, int BX, int S>
void fill_stream(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_stream<NS, T, 0, BX, S>;
    e.launch[prec][1][slot] = &launch_stream<NS, T, 1, BX, S>;
    e.launch[prec][2][slot] = &launch_stream<NS, T, 2, BX, S>;
    e.launch[prec][3][slot] = &launch_stream<NS, T, 3, BX, S>;
    e.launch[prec][4][slot] = &launch_stream<NS, T, 4, BX, S>;
    e.sched_name[prec][slot] = "stream cp.async block " + std::to_string(BX) + " stages " + std::to_string(S);
    for (int v = 0; v < 5; ++v)
        if (e.best[prec][v] == 0 && v != ACS_ORIGINAL) e.best[prec][v] = slot;
}

}  // namespace acs
