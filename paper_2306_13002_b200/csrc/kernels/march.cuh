// march.cuh — the TMA "marching tile" skeleton (the backend's TILED schedule).
//
// A CTA owns a tile of the inner loop(s) — TX points of the innermost loop
// (and TY of the middle loop for 3-D nests) — and marches along the outermost
// loop over a chunk.  Every array the nest LOADS (and never stores) is staged
// in shared memory by the Tensor Memory Accelerator: per march step, one
// cp.async.bulk.tensor box per array holding exactly the elements the tile's
// points read at that plane (the stencil halo of the tile, all D3Q19
// distribution components, ...).  Boxes live in a ring of D = span + PF slots
// guarded by mbarriers, so PF planes are always in flight ahead of the
// compute — memory-level parallelism no longer depends on register pressure —
// and each plane of a stencil array is fetched once per tile however many
// k-neighbours read it (the paper's "common loads held on chip", applied
// across loop iterations; bulk-load order realised as one TMA per array).
//
// The generated body of the requested form (original or reference-emitted)
// is unchanged: ld<ARR, o...>() becomes an LDS from the ring,
// data-dependent ldx<ARR>(...) is served from the staged box when the index
// lands inside it and from global memory otherwise (always correct), and
// stores go straight to HBM, coalesced along the innermost loop.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <utility>

#include "../acs_device.cuh"
#include "../registry.hpp"
#include "../tma.cuh"

namespace acs {

// LAYOUT 0: row-major (reference layout, optionally with padded pitches);
// LAYOUT 1: trailing subscript slowest (D3Q19 q-major SoA).
template <class NS, class T, int LAYOUT, int TX, int TY>
struct MarchPlan {
    static constexpr int NL = NS::NLOOP;
    static constexpr int X = NL - 1;   // loop index of the innermost loop (tile x)
    static constexpr int Y = NL == 3 ? 1 : -9;

    static constexpr int esize(int a) { return NS::is_int(a) ? 4 : (int)sizeof(T); }
    // LAYOUT 1 applies to arrays whose trailing subscript is a component index
    // (absolute constant, e.g. the D3Q19 q): that subscript is the slowest.
    static constexpr bool soa(int a) { return LAYOUT == 1 && NS::ndim(a) >= 2 && NS::sig(a, NS::ndim(a) - 1) == -1; }
    static constexpr int pos_of_dim(int a, int d) {
        const int nd = NS::ndim(a);
        if (soa(a)) return d < nd - 1 ? nd - 2 - d : nd - 1;
        return nd - 1 - d;
    }
    static constexpr int march_pos(int a) {
        for (int p = 0; p < NS::ndim(a); ++p)
            if (NS::ld_sig(a, p) == 0) return p;
        return -1;
    }
    static constexpr bool staged(int a) { return NS::stageable(a); }
    static constexpr bool on_ring(int a) { return staged(a) && march_pos(a) >= 0; }
    static constexpr bool is_static(int a) { return staged(a) && march_pos(a) < 0; }
    static constexpr int span(int a) {
        const int mp = march_pos(a);
        return mp < 0 ? 0 : NS::ld_hi(a, mp) - NS::ld_lo(a, mp) + 1;
    }
    static constexpr int maxspan() {
        int m = 0;
        for (int a = 0; a < NS::NARR; ++a)
            if (on_ring(a) && span(a) > m) m = span(a);
        return m;
    }
    static constexpr int raw_extent(int a, int p) {
        const int s = NS::ld_sig(a, p);
        const int w = NS::ld_hi(a, p) - NS::ld_lo(a, p);
        if (s == 0) return 1;
        if (s == X) return TX + w;
        if (s == Y) return TY + w;
        return w + 1;
    }
    // TMA (measured on B200: an unaligned start raises "illegal instruction"):
    // the innermost box row must start on a 16-byte boundary and span a
    // multiple of 16 bytes.  The box start is aligned down by a per-array
    // shift (same for every CTA, see MarchMem::sh), so the innermost extent
    // reserves q-1 extra elements.
    static constexpr int xq(int a) { return 16 / esize(a); }
    static constexpr bool inner_is_x(int a) { return NS::ld_sig(a, pos_of_dim(a, 0)) == X; }
    static constexpr int extent(int a, int p) {
        const int e = raw_extent(a, p);
        if (p != pos_of_dim(a, 0)) return e;
        const int q = xq(a);
        const int need = inner_is_x(a) ? e + q - 1 : e;
        return (need + q - 1) / q * q;
    }
    static constexpr int bstride(int a, int p) {   // element stride of position p inside the box
        int st = 1;
        for (int d = 0; d < NS::ndim(a); ++d) {
            if (pos_of_dim(a, d) == p) return st;
            st *= extent(a, pos_of_dim(a, d));
        }
        return st;
    }
    static constexpr int box_bytes(int a) {
        int n = esize(a);
        for (int p = 0; p < NS::ndim(a); ++p) n *= extent(a, p);
        return n;
    }
    static constexpr int align128(int b) { return (b + 127) / 128 * 128; }
    static constexpr int ring_off(int a) {   // byte offset of array a inside one ring slot
        int o = 0;
        for (int b = 0; b < a; ++b)
            if (on_ring(b)) o += align128(box_bytes(b));
        return o;
    }
    static constexpr int slot_bytes() { return ring_off(NS::NARR); }
    static constexpr int slot_tx() {
        int t = 0;
        for (int a = 0; a < NS::NARR; ++a)
            if (on_ring(a)) t += box_bytes(a);
        return t;
    }
    static constexpr int static_off(int a) {
        int o = 0;
        for (int b = 0; b < a; ++b)
            if (is_static(b)) o += align128(box_bytes(b));
        return o;
    }
    static constexpr int static_bytes() { return static_off(NS::NARR); }
    static constexpr int static_tx() {
        int t = 0;
        for (int a = 0; a < NS::NARR; ++a)
            if (is_static(a)) t += box_bytes(a);
        return t;
    }
    static constexpr bool usable() {
        if (maxspan() < 1) return false;
        for (int a = 0; a < NS::NARR; ++a)
            if (staged(a))
                for (int p = 0; p < NS::ndim(a); ++p) {
                    if (extent(a, p) > 256) return false;
                    const int s = NS::ld_sig(a, p);
                    if (s != -1 && s != 0 && s != X && s != Y) return false;
                }
        return true;
    }
};

template <class NS>
struct TmaMaps {
    CUtensorMap m[NS::NARR];
};

// per-CTA state a body's memory policy needs
template <class NS, class T, int LAYOUT, int TX, int TY, int PF>
struct MarchMem {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY>;
    static constexpr int D = P::maxspan() + PF;
    NaiveMem<NS, T, false> g;
    const unsigned char* ring;     // slot 0
    const unsigned char* stat;     // static boxes
    int newest;                    // ring slot of the newest bundle this step needs
    int lx, ly;                    // this thread's position inside the tile
    int k;                         // current march coordinate
    int orgx, orgy;
    int sh[NS::NARR];              // innermost-box alignment shift per array (elements)

    template <int ARR>
    using elem_t = typename NaiveMem<NS, T, false>::template elem_t<ARR>;

    template <int ARR>
    __device__ __forceinline__ const elem_t<ARR>* box_base(int slot_delta) const {
        if constexpr (P::on_ring(ARR)) {
            int slot = newest + slot_delta;
            slot = slot >= D ? slot - D : slot;
            return reinterpret_cast<const elem_t<ARR>*>(ring + slot * P::slot_bytes() + P::ring_off(ARR));
        } else {
            return reinterpret_cast<const elem_t<ARR>*>(stat + P::static_off(ARR));
        }
    }

    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const {
        if constexpr (P::staged(ARR)) {
            constexpr int off[sizeof...(O)] = {O...};
            int idx = 0;
            int delta = D;   // slot delta relative to `newest`, kept in [0, D) by box_base
#pragma unroll
            for (int p = 0; p < (int)sizeof...(O); ++p) {
                const int s = NS::ld_sig(ARR, p);
                const int l = off[p] - NS::ld_lo(ARR, p);
                if (s == 0) delta = D + off[p] - NS::ld_hi(ARR, p);
                else if (s == P::X) idx += (lx + l + sh[ARR]) * P::bstride(ARR, p);
                else if (s == P::Y) idx += (ly + l) * P::bstride(ARR, p);
                else idx += l * P::bstride(ARR, p);
            }
            if (delta >= D) delta -= D;
            return box_base<ARR>(delta)[idx];
        } else {
            return g.template ld<ARR, O...>();
        }
    }

    // out-of-box dynamic index: rare (e.g. advec's clamp at the domain edge),
    // kept out of line so the in-box path stays a few integer ops + one LDS
    template <int ARR, class... I>
    __device__ __noinline__ elem_t<ARR> ldx_global(I... ii) const { return g.template ldx<ARR>(ii...); }

    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... ii) const {
        if constexpr (P::staged(ARR)) {
            const int v[sizeof...(I)] = {(int)ii...};
            int idx = 0, delta = 0;
            unsigned out = 0;
#pragma unroll
            for (int p = 0; p < (int)sizeof...(I); ++p) {
                const int s = NS::ld_sig(ARR, p);
                const int lo = NS::ld_lo(ARR, p);
                if (s == 0) {
                    const int d = v[p] - k;
                    out |= (unsigned)(d - lo) > (unsigned)(NS::ld_hi(ARR, p) - lo);
                    delta = D + d - NS::ld_hi(ARR, p);
                } else {
                    const int l = v[p] - lo - (s == P::X ? orgx : (s == P::Y ? orgy : 0));
                    out |= (unsigned)l >= (unsigned)P::raw_extent(ARR, p);
                    idx += (l + (s == P::X ? sh[ARR] : 0)) * P::bstride(ARR, p);
                }
            }
            if (__builtin_expect(out == 0, 1)) {
                if (delta >= D) delta -= D;
                return box_base<ARR>(delta)[idx];
            }
            return ldx_global<ARR>(ii...);
        } else {
            return g.template ldx<ARR>(ii...);
        }
    }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const { g.template st<ARR, O...>(v); }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const { g.template stx<ARR>(args...); }
};

template <class P, class NS>
__host__ __device__ constexpr int xshift(int a, int orgx) {
    if (!P::inner_is_x(a)) return 0;
    const int q = P::xq(a);
    const int v = orgx + NS::ld_lo(a, P::pos_of_dim(a, 0));
    return ((v % q) + q) % q;
}

template <class P, class NS, int A>
__device__ __forceinline__ void march_issue(unsigned char* slot_base, const TmaMaps<NS>& maps, uint64_t* bar,
                                            int plane_base, int orgx, int orgy, bool want_static,
                                            unsigned char* stat) {
    if constexpr (A < NS::NARR) {
        constexpr bool take = P::on_ring(A) || P::is_static(A);
        if constexpr (take) {
            if (P::on_ring(A) != want_static) {   // ring boxes per bundle, static boxes once
                int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
                for (int d = 0; d < NS::ndim(A); ++d) {
                    const int p = P::pos_of_dim(A, d);
                    const int s = NS::ld_sig(A, p);
                    if (s == 0) c[d] = plane_base + NS::ld_hi(A, p);
                    else if (s == P::X) c[d] = orgx + NS::ld_lo(A, p) - (d == 0 ? xshift<P, NS>(A, orgx) : 0);
                    else if (s == P::Y) c[d] = orgy + NS::ld_lo(A, p);
                    else c[d] = NS::ld_lo(A, p);
                }
                unsigned char* dst = P::on_ring(A) ? slot_base + P::ring_off(A) : stat + P::static_off(A);
                tma_load<NS::ndim(A)>(dst, &maps.m[A], c, bar);
            }
        }
        march_issue<P, NS, A + 1>(slot_base, maps, bar, plane_base, orgx, orgy, want_static, stat);
    }
}

// TX x TY points per tile, BX x BY threads: each thread computes (TX/BX) x (TY/BY)
// points per march step, amortising the step's barrier / mbarrier wait.
template <class NS, class T, int FORM, int LAYOUT, int TX, int TY, int BX, int BY, int PF>
__global__ void __launch_bounds__(BX* BY) march_kernel(const __grid_constant__ KernelArgs<NS> args,
                                                       const __grid_constant__ TmaMaps<NS> maps, int kchunk) {
    static_assert(TX % BX == 0 && TY % BY == 0, "tile must be a multiple of the block");
    using P = MarchPlan<NS, T, LAYOUT, TX, TY>;
    using M = MarchMem<NS, T, LAYOUT, TX, TY, PF>;
    constexpr int D = M::D;
    constexpr int MS = P::maxspan();
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem;
    unsigned char* stat = smem + D * P::slot_bytes();
    uint64_t* bars = reinterpret_cast<uint64_t*>(stat + P::static_bytes());   // D ring + 1 static

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * BX + tx;
    const int orgx = args.lo[P::X] + blockIdx.x * TX;
    const int orgy = NS::NLOOP == 3 ? args.lo[1] + blockIdx.y * TY : 0;
    const int kb = args.lo[0] + blockIdx.z * kchunk;
    const int ke = min(kb + kchunk, args.hi[0]);
    const int ns = ke - kb;
    const int nb = ns + MS - 1;   // bundles this chunk consumes

    if (tid == 0) {
        for (int s = 0; s <= D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        if constexpr (P::static_tx() > 0) {
            mbar_expect_tx(&bars[D], P::static_tx());
            march_issue<P, NS, 0>(nullptr, maps, &bars[D], 0, orgx, orgy, true, stat);
        }
        for (int B = 0; B < D - 1 && B < nb; ++B) {
            mbar_expect_tx(&bars[B % D], P::slot_tx());
            march_issue<P, NS, 0>(ring + (B % D) * P::slot_bytes(), maps, &bars[B % D], kb + B - (MS - 1), orgx,
                                  orgy, false, stat);
        }
    }
    if constexpr (P::static_tx() > 0) mbar_wait(&bars[D], 0);
    // TMA transfers complete in any order: step 0 needs bundles 0 .. MS-1, the
    // loop below waits only for the newest bundle of each step.
    for (int B = 0; B < MS - 1 && B < nb; ++B) mbar_wait(&bars[B % D], 0);

    int pt[NS::NLOOP];
    M m{NaiveMem<NS, T, false>{args, pt}, ring, stat, 0, tx, ty, 0, orgx, orgy, {}};
#pragma unroll
    for (int a = 0; a < NS::NARR; ++a) m.sh[a] = xshift<P, NS>(a, orgx);

    for (int s = 0; s < ns; ++s) {
        __syncthreads();   // every thread is done with step s-1: its oldest slot is free
        if (tid == 0) {
            const int B = s + D - 1;
            if (B < nb) {
                fence_proxy_async();
                mbar_expect_tx(&bars[B % D], P::slot_tx());
                march_issue<P, NS, 0>(ring + (B % D) * P::slot_bytes(), maps, &bars[B % D], kb + B - (MS - 1),
                                      orgx, orgy, false, stat);
            }
        }
        const int Bw = s + MS - 1;
        mbar_wait(&bars[Bw % D], (uint32_t)((Bw / D) & 1));
        pt[0] = kb + s;
        m.k = kb + s;
        m.newest = Bw % D;
#pragma unroll
        for (int ry = 0; ry < TY / BY; ++ry) {
#pragma unroll
            for (int rx = 0; rx < TX / BX; ++rx) {
                m.lx = tx + rx * BX;
                m.ly = ty + ry * BY;
                const int x = orgx + m.lx, y = orgy + m.ly;
                if (x < args.hi[P::X] && (NS::NLOOP < 3 || y < args.hi[1])) {
                    pt[P::X] = x;
                    if constexpr (NS::NLOOP == 3) pt[1] = y;
                    NS::template body<FORM>(m, args.s, pt);
                }
            }
        }
    }
}

// ---- host launcher -----------------------------------------------------------

inline bool acs_debug() {
    static const bool on = std::getenv("ACS_DEBUG") != nullptr;
    return on;
}
#define ACS_TMA_FAIL(msg)                                                                   \
    do {                                                                                    \
        if (acs_debug()) std::fprintf(stderr, "[acs] TMA fallback (%s): %s\n", NS::array_names[a], msg); \
        return false;                                                                       \
    } while (0)

template <class NS, class T, int LAYOUT, int TX, int TY>
bool encode_maps(const LaunchReq& r, TmaMaps<NS>& maps) {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY>;
    EncodeTiledFn enc = tma_encoder();
    if (!enc) {
        if (acs_debug()) std::fprintf(stderr, "[acs] no cuTensorMapEncodeTiled entry point\n");
        return false;
    }
    for (int a = 0; a < NS::NARR; ++a) {
        if (!P::staged(a)) continue;
        const acs_array* d = nullptr;
        for (int i = 0; i < r.n_arrays; ++i)
            if (std::strcmp(r.arrays[i].name, NS::array_names[a]) == 0) d = &r.arrays[i];
        if (!d) ACS_TMA_FAIL("missing");
        const int nd = d->ndim;
        long long st[8];
        bool rm = true;
        for (int p = 0; p < nd; ++p) rm = rm && d->strides[p] == 0;
        long long acc = 1;
        for (int p = nd - 1; p >= 0; --p) {
            st[p] = rm ? acc : d->strides[p];
            acc *= d->dims[p];
        }
        const int es = P::esize(a);
        if (reinterpret_cast<uintptr_t>(d->data) % 16 != 0) ACS_TMA_FAIL("base not 16-byte aligned");
        cuuint64_t gdim[5], gstr[4];
        cuuint32_t box[5], estr[5];
        long long prev = 0;
        for (int dd = 0; dd < nd; ++dd) {
            const int p = P::pos_of_dim(a, dd);
            if (dd == 0 && st[p] != 1) ACS_TMA_FAIL("innermost dim not contiguous");
            if (dd > 0) {
                if (st[p] <= prev || (st[p] * es) % 16 != 0) ACS_TMA_FAIL("stride order / 16-byte multiple");
                gstr[dd - 1] = (cuuint64_t)(st[p] * es);
            }
            prev = st[p];
            gdim[dd] = (cuuint64_t)d->dims[p];
            box[dd] = (cuuint32_t)P::extent(a, p);
            estr[dd] = 1;
        }
        const CUtensorMapDataType dt = NS::is_int(a) ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                       : sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                        : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        CUresult e = enc(&maps.m[a], dt, (cuuint32_t)nd, d->data, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (acs_debug()) {
            std::fprintf(stderr, "[acs] map %s rank %d base %p", NS::array_names[a], nd, d->data);
            for (int dd = 0; dd < nd; ++dd)
                std::fprintf(stderr, " | d%d dim %llu box %u stride %llu", dd, (unsigned long long)gdim[dd], box[dd],
                             dd ? (unsigned long long)gstr[dd - 1] : 0ULL);
            std::fprintf(stderr, " | ring_off %d slot %d D %d\n", P::ring_off(a), P::slot_bytes(), P::maxspan());
        }
        if (e != CUDA_SUCCESS) {
            if (acs_debug())
                std::fprintf(stderr, "[acs] cuTensorMapEncodeTiled(%s) = %d rank %d box %u %u %u %u\n", NS::array_names[a],
                             (int)e, nd, box[0], nd > 1 ? box[1] : 0, nd > 2 ? box[2] : 0, nd > 3 ? box[3] : 0);
            return false;
        }
    }
    return true;
}

template <class NS, class T, int FORM, int LAYOUT, int TX, int TY, int BX, int BY, int PF>
acs_status launch_march(const LaunchReq& r) {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY>;
    static_assert(P::usable(), "march skeleton: nest not stageable");
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    TmaMaps<NS> maps;
    std::memset(&maps, 0, sizeof maps);
    if (!encode_maps<NS, T, LAYOUT, TX, TY>(r, maps)) {
        // layout the TMA cannot describe (unaligned base / pitch): same
        // numerics through the global-memory skeleton
        return launch_naive<NS, T, FORM>(r);
    }
    constexpr int D = P::maxspan() + PF;
    constexpr int smem = D * P::slot_bytes() + P::static_bytes() + (D + 1) * 8;
    auto kern = march_kernel<NS, T, FORM, LAYOUT, TX, TY, BX, BY, PF>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    constexpr int NL = NS::NLOOP;
    const long long nx = ka.hi[NL - 1] - ka.lo[NL - 1];
    const long long ny = NL == 3 ? ka.hi[1] - ka.lo[1] : 1;
    const long long nz = ka.hi[0] - ka.lo[0];
    const long long tiles = ((nx + TX - 1) / TX) * (NL == 3 ? (ny + TY - 1) / TY : 1);
    // ~8 waves of CTAs; chunks long enough to amortise the (span-1)-plane prologue
    const long long want = (148LL * 4 * 8 + tiles - 1) / tiles;
    long long kchunk = (nz + want - 1) / want;
    const long long minch = 4LL * (P::maxspan() > 1 ? P::maxspan() : 2);
    if (kchunk < minch) kchunk = minch;
    if (kchunk > nz) kchunk = nz;
    const long long chunks = (nz + kchunk - 1) / kchunk;
    dim3 grid((unsigned)((nx + TX - 1) / TX), (unsigned)(NL == 3 ? (ny + TY - 1) / TY : 1), (unsigned)chunks);
    kern<<<grid, dim3(BX, BY, 1), smem, r.stream>>>(ka, maps, (int)kchunk);
    return check_launch("march");
}

template <class NS, class T, int LAYOUT, int TX, int TY, int BX, int BY, int PF>
void fill_march(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_march<NS, T, 0, LAYOUT, TX, TY, BX, BY, PF>;
    e.launch[prec][1][slot] = &launch_march<NS, T, 1, LAYOUT, TX, TY, BX, BY, PF>;
    e.launch[prec][2][slot] = &launch_march<NS, T, 2, LAYOUT, TX, TY, BX, BY, PF>;
    e.launch[prec][3][slot] = &launch_march<NS, T, 3, LAYOUT, TX, TY, BX, BY, PF>;
    e.launch[prec][4][slot] = &launch_march<NS, T, 4, LAYOUT, TX, TY, BX, BY, PF>;
    e.sched_name[prec][slot] = "march tile " + std::to_string(TX) + "x" + std::to_string(TY) + " block " +
                               std::to_string(BX) + "x" + std::to_string(BY) + " pf " + std::to_string(PF);
    for (int v = 0; v < 5; ++v)
        if (e.best[prec][v] == 0 && v != ACS_ORIGINAL) e.best[prec][v] = slot;
}

}  // namespace acs
