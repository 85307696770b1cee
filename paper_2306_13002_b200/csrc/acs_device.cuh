// acs_device.cuh — device-side building blocks shared by every nest skeleton.
//
// A generated body (csrc/gen/<nest>.cuh, from paper_2306_13002_b200/lowering.py)
// asks its memory policy `m` for array elements:
//     m.template ld<ARR, o0, o1, ...>()      subscript p = point[sig(ARR,p)] + o_p
//                                             (or the constant o_p when sig = -1)
//     m.template ldx<ARR>(i0, i1, ...)        data-dependent absolute subscripts
//     m.template st<ARR, o...>(v) / stx<ARR>(i..., v)
// The policy decides where the element lives.  NaiveMem (here) is plain global
// memory addressed through per-array element strides — the reference layout
// (ArrayBuf::flat, proj/src/interp.cpp:10-22) or a backend layout such as the
// D3Q19 q-major SoA.  Tiled skeletons (csrc/kernels/*.cuh) wrap it.
#pragma once

#include <cstdint>
#include <type_traits>

namespace acs {

constexpr int kMaxArrays = 24;

struct ArrayView {
    char* base;
    long long stride[8];   // element strides per subscript position
};

// Slab sharding (owner computes, write-through to every holder): a store to
// global plane g of a sharded array is also written straight into the lower
// neighbour's buffer when g < lo_thr and into the upper neighbour's when
// g >= hi_thr (peer memory over NVLink, or the same device).  dlo/dhi are the
// element offsets from this rank's buffer index to the neighbour's.
template <int NARR>
struct ShardArgs {
    int enabled;
    long long origin;    // global coordinate of local index 0 along subscript 0
    long long lo_thr, hi_thr;
    char* peer_lo[NARR];
    char* peer_hi[NARR];
    long long dlo[NARR], dhi[NARR];
};

template <class NS>
struct KernelArgs {
    ArrayView arr[NS::NARR];
    typename NS::Scalars s;
    int lo[NS::NLOOP];
    int hi[NS::NLOOP];
    ShardArgs<NS::NARR> sh;
};

// ---- raw access primitives ------------------------------------------------

template <class T>
__device__ __forceinline__ T ld_plain(const T* p) { return *p; }

template <class T>
__device__ __forceinline__ T ld_ro(const T* p) { return __ldg(p); }

// One real global load that the compiler may neither merge with another,
// drop, nor move across other memory operations: the ORIGINAL form's
// as-written load (a directive compiler without alias information).
__device__ __forceinline__ double ld_asis(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float ld_asis(const float* p) {
    float v;
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_asis(const int* p) {
    int v;
    asm volatile("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_asis(double* p, double v) {
    asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_asis(float* p, float v) {
    asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_asis(int* p, int v) {
    asm volatile("st.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- the naive (global-memory) policy --------------------------------------

template <class NS, class T, bool ASIS>
struct NaiveMem {
    const KernelArgs<NS>& a;
    const int* pt;

    template <int ARR>
    using elem_t = std::conditional_t<NS::is_int(ARR), int, T>;

    template <int ARR, int... O>
    __device__ __forceinline__ long long static_index() const {
        constexpr int offs[sizeof...(O)] = {O...};
        long long idx = 0;
#pragma unroll
        for (int p = 0; p < (int)sizeof...(O); ++p) {
            const int s = NS::sig(ARR, p);
            const long long v = (s >= 0 ? (long long)pt[s < 0 ? 0 : s] : 0LL) + offs[p];
            idx += v * a.arr[ARR].stride[p];
        }
        return idx;
    }

    template <int ARR, class... I>
    __device__ __forceinline__ long long dyn_index(I... idx) const {
        const long long v[sizeof...(I)] = {(long long)idx...};
        long long r = 0;
#pragma unroll
        for (int p = 0; p < (int)sizeof...(I); ++p) r += v[p] * a.arr[ARR].stride[p];
        return r;
    }

    template <int ARR>
    __device__ __forceinline__ elem_t<ARR>* ptr(long long idx) const {
        return reinterpret_cast<elem_t<ARR>*>(a.arr[ARR].base) + idx;
    }

    template <int ARR>
    __device__ __forceinline__ elem_t<ARR> load_at(long long idx) const {
        if constexpr (ASIS) return ld_asis(ptr<ARR>(idx));
        else if constexpr (NS::readonly(ARR)) return ld_ro(ptr<ARR>(idx));
        else return ld_plain(ptr<ARR>(idx));
    }
    template <int ARR>
    __device__ __forceinline__ void store_at(long long idx, elem_t<ARR> v) const {
        if constexpr (ASIS) st_asis(ptr<ARR>(idx), v);
        else *ptr<ARR>(idx) = v;
    }

    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const { return load_at<ARR>(static_index<ARR, O...>()); }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... idx) const { return load_at<ARR>(dyn_index<ARR>(idx...)); }
    // data-dependent index the lowering proved to lie in the load's value set
    // (every candidate affine in the loop variables): same element as ldx
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx_in(I... idx) const { return ldx<ARR>(idx...); }
    // write-through of a store to the neighbours that hold plane l0 (sharded launches)
    template <int ARR>
    __device__ __forceinline__ void forward(long long idx, long long l0, elem_t<ARR> v) const {
        const long long g = l0 + a.sh.origin;
        if (g < a.sh.lo_thr && a.sh.peer_lo[ARR])
            *(reinterpret_cast<elem_t<ARR>*>(a.sh.peer_lo[ARR]) + idx + a.sh.dlo[ARR]) = v;
        if (g >= a.sh.hi_thr && a.sh.peer_hi[ARR])
            *(reinterpret_cast<elem_t<ARR>*>(a.sh.peer_hi[ARR]) + idx + a.sh.dhi[ARR]) = v;
    }

    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const {
        const long long idx = static_index<ARR, O...>();
        store_at<ARR>(idx, v);
        if constexpr (NS::sig(ARR, 0) == 0) {
            if (a.sh.enabled) {
                constexpr int off[sizeof...(O)] = {O...};
                forward<ARR>(idx, (long long)pt[0] + off[0], v);
            }
        }
    }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const {
        // last argument is the value; the rest are subscripts
        stx_impl<ARR>(args...);
    }

  private:
    template <int ARR, class I0, class V>
    __device__ __forceinline__ void stx_at(long long idx, I0 i0, V v) const {
        store_at<ARR>(idx, v);
        if (a.sh.enabled) forward<ARR>(idx, (long long)i0, v);
    }
    template <int ARR, class I0, class V>
    __device__ __forceinline__ void stx_impl(I0 i0, V v) const { stx_at<ARR>(dyn_index<ARR>(i0), i0, v); }
    template <int ARR, class I0, class I1, class V>
    __device__ __forceinline__ void stx_impl(I0 i0, I1 i1, V v) const { stx_at<ARR>(dyn_index<ARR>(i0, i1), i0, v); }
    template <int ARR, class I0, class I1, class I2, class V>
    __device__ __forceinline__ void stx_impl(I0 i0, I1 i1, I2 i2, V v) const {
        stx_at<ARR>(dyn_index<ARR>(i0, i1, i2), i0, v);
    }
    template <int ARR, class I0, class I1, class I2, class I3, class V>
    __device__ __forceinline__ void stx_impl(I0 i0, I1 i1, I2 i2, I3 i3, V v) const {
        stx_at<ARR>(dyn_index<ARR>(i0, i1, i2, i3), i0, v);
    }
};

// One thread per point of the marked loop nest: innermost loop on x, the next
// on y, the outermost (3-D nests) on z — the gang/worker/vector mapping of the
// nest's own directives.
template <class NS, class T, int FORM, bool ASIS, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) naive_kernel(const __grid_constant__ KernelArgs<NS> args) {
    constexpr int NL = NS::NLOOP;
    int pt[NL];
    const int x = args.lo[NL - 1] + (int)(blockIdx.x * blockDim.x + threadIdx.x);
    if (x >= args.hi[NL - 1]) return;
    pt[NL - 1] = x;
    if constexpr (NL >= 2) {
        const int y = args.lo[NL - 2] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
        if (y >= args.hi[NL - 2]) return;
        pt[NL - 2] = y;
    }
    if constexpr (NL >= 3) {
        const int z = args.lo[NL - 3] + (int)blockIdx.z;
        if (z >= args.hi[NL - 3]) return;
        pt[NL - 3] = z;
    }
    NaiveMem<NS, T, ASIS> m{args, pt};
    NS::template body<FORM>(m, args.s, pt);
    // sharded launch: this thread's write-through stores to peer memory are
    // performed system-wide before the kernel retires (the signal kernel that
    // follows on the stream then releases the step flag)
    if (args.sh.enabled) __threadfence_system();
}

// R points per thread along the innermost loop, strided by the block width
// (each r-slice of a warp is still one coalesced row segment): R
// independent bodies per thread, so the read-only (ld.global.nc) loads of
// all R points can be in flight together — more bytes in flight per SM for
// point-local streaming nests (ideal_gas, calc3) at the same occupancy.
template <class NS, class T, int FORM, int R>
__global__ void __launch_bounds__(256) naive_multi_kernel(const __grid_constant__ KernelArgs<NS> args) {
    constexpr int NL = NS::NLOOP;
    int pt[NL];
    if constexpr (NL >= 2) {
        const int y = args.lo[NL - 2] + (int)(blockIdx.y * blockDim.y + threadIdx.y);
        if (y >= args.hi[NL - 2]) return;
        pt[NL - 2] = y;
    }
    if constexpr (NL >= 3) {
        const int z = args.lo[NL - 3] + (int)blockIdx.z;
        if (z >= args.hi[NL - 3]) return;
        pt[NL - 3] = z;
    }
    const int x0 = args.lo[NL - 1] + (int)(blockIdx.x * blockDim.x * R + threadIdx.x);
    NaiveMem<NS, T, FORM == 0> m{args, pt};
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int x = x0 + r * (int)blockDim.x;
        if (x < args.hi[NL - 1]) {
            pt[NL - 1] = x;
            NS::template body<FORM>(m, args.s, pt);
        }
    }
    if (args.sh.enabled) __threadfence_system();
}

}  // namespace acs
