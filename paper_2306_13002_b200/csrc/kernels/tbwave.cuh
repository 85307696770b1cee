// tbwave.cuh — temporal blocking of a 3-level leapfrog star stencil of
// radius 2 (seismic wave4: un = f(u, up, vel2); the time loop rotates
// up <- u <- un), two time steps per launch.
//
// The kernels/tblock.cuh scheme (TMA plane ring, register k-columns, the
// step-1 field in a shared ring, one barrier per plane) with what the
// leapfrog adds:
//   * per march plane the TMA brings three boxes into one ring slot: u with a
//     4-cell halo (step 1 on the 2-cell extended tile reads ±2), and up and
//     vel2 on the extended tile's rows (x from u's 16-byte aligned origin);
//   * step 1 (plane p, extended (TX+4) x (TY+4) tile) writes S1 = un to the
//     shared ring AND, on the own tile, to HBM: after two steps the state is
//     up = S1, u = S2, so S1 is output too;
//   * step 2 (plane p-2, the tile) reads S1 from the ring / the thread's own
//     S1 k-column, its "up" is u at that plane (still in the u k-column) and
//     vel2 comes from a per-cell register queue; it writes S2 to a FOURTH
//     buffer `un2`: the rotation's free buffer (up) is still read by the
//     neighbour tiles' step 1, so writing S2 there would race;
//   * S1 outside the iteration space (the fixed 2-cell boundary and the
//     boundary planes) is the value the step-by-step loop would read there:
//     the `un` buffer's, loaded from HBM for those cells only.
// A CTA of TX x TY/NY threads owns a TX x TY tile, NY cells of a column per
// thread (y neighbours between them from registers); threads 0..NR-1 also own
// one cell of the 2-wide halo ring of the extended tile.  The plane loop is
// unrolled by 5 (the k-column length): ring slots, queue positions and the
// S1 ring slot are compile-time.  HBM per two steps: u, up, vel2 read once,
// un and un2 written once = 20 B/point (fp32) instead of 32.  Same generated
// body as every skeleton: bit-exact against two step-by-step launches
// (precondition: every rotating buffer carries the same fixed boundary).
// Measured on B200 (profiles/r02_wave4_tb2.md): with per-cell predicates and
// plane pointers hoisted out of the march (139 -> 108 instructions per point
// per two steps) it runs at 1.02-1.04x of two tuned single-step launches;
// the 2-wide halo ring (40 % extra step-1 work) keeps it issue-bound.
#pragma once

#include <cstdlib>

#include "../acs_device.cuh"
#include "../registry.hpp"
#include "../tma.cuh"
#include "tblock.cuh"

namespace acs {

template <class NS, int IU, int IUP, int IUN, int IV>
struct TwPlan {
    static constexpr bool usable() {
        if (NS::NARR != 4 || NS::NLOOP != 3 || NS::has_dynamic_index) return false;
        if (!NS::readonly(IU) || !NS::readonly(IUP) || !NS::readonly(IV) || NS::readonly(IUN)) return false;
        for (int p = 0; p < 3; ++p) {
            if (NS::ld_sig(IU, p) != p || NS::ld_lo(IU, p) < -2 || NS::ld_hi(IU, p) > 2) return false;
            if (NS::ld_lo(IUP, p) != 0 || NS::ld_hi(IUP, p) != 0 || NS::ld_lo(IV, p) != 0 || NS::ld_hi(IV, p) != 0)
                return false;
        }
        if (NS::NSROW != 1 || NS::srow_arr(0) != IUN) return false;
        for (int p = 0; p < 3; ++p)
            if (NS::srow_off(0, p) != 0) return false;
        for (int r = 0; r < NS::NROW; ++r)
            if (NS::row_arr(r) == IU && NS::row_off(r, 0) != 0 &&
                (NS::row_off(r, 1) != 0 || NS::row_xlo(r) != 0 || NS::row_xhi(r) != 0))
                return false;
        return true;
    }
};

// one cell of one step: the stencil array's k-column q[0..4] (planes k-2..k+2)
// and the thread's other cells' centres yc[] from registers, the other in-plane
// neighbours from shared memory at `a` (row stride RS elements), the point-local
// operands as values; the store lands in *out
template <class T, int RS, int NY, int IU, int IUP, int IV>
struct TwMem {
    unsigned a;
    const T* q;
    const T* yc;
    int c;
    T up, vel;
    T* out;
    template <int ARR>
    using elem_t = T;
    template <int ARR, int... O>
    __device__ __forceinline__ T ld() const {
        constexpr int off[sizeof...(O)] = {O...};
        if constexpr (ARR == IU) {
            if constexpr (off[1] == 0 && off[2] == 0) {
                return q[off[0] + 2];
            } else {
                static_assert(off[0] == 0, "tbw: off-plane loads are centre cells (a star stencil)");
                if constexpr (off[2] == 0)
                    if (c + off[1] >= 0 && c + off[1] < NY) return yc[c + off[1]];
                constexpr int o = (off[1] * RS + off[2]) * (int)sizeof(T);
                return tb_lds(a + (unsigned)o, T(0));
            }
        } else if constexpr (ARR == IUP) {
            return up;
        } else {
            static_assert(ARR == IV, "tbw: unexpected array");
            return vel;
        }
    }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(T v) const {
        *out = v;
    }
    template <int ARR, class... I>
    __device__ __forceinline__ T ldx(I...) const { return T(0); }
    template <int ARR, class... I>
    __device__ __forceinline__ T ldx_in(I...) const { return T(0); }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A...) const {}
};

template <int TX, int TY, int NY, class T>
struct TwGeom {
    static constexpr int UX = TX + 8, UY = TY + 8;      // u box (4-cell halo)
    static constexpr int IX = TX + 4, IY = TY + 4;      // extended tile: up / vel2 boxes, S1 plane
    static constexpr int D = 5;                         // ring planes (PF = 2 in flight)
    static constexpr int NT = TX * TY / NY;
    static constexpr int NR = IX * IY - TX * TY;        // 2-wide halo ring of the extended tile
    static constexpr unsigned r128(unsigned b) { return (b + 127) / 128 * 128; }
    // u box UX x UY; up / vel2 boxes UX x IY (the extended tile's rows, u's x origin)
    static constexpr unsigned UB = UX * UY * sizeof(T), VB = UX * IY * sizeof(T), EB = IX * IY * sizeof(T);
    static constexpr unsigned OFF_UP = r128(UB), OFF_V = OFF_UP + r128(VB);
    static constexpr unsigned SLOT = OFF_V + r128(VB);
    static constexpr unsigned SPLANE = r128(EB);
    static constexpr int smem = D * SLOT + 5 * SPLANE + D * 8;
    static_assert(NR <= NT, "tbw: the halo ring needs at most one cell per thread");
    static_assert(TY % NY == 0, "tbw: NY divides the tile height");
    static_assert((UX * (int)sizeof(T)) % 16 == 0 && (IX * (int)sizeof(T)) % 16 == 0, "tbw: TMA rows");
};

struct TwMaps {
    CUtensorMap u, up, vel;
};

template <class NS, class T, int FORM, int IU, int IUP, int IUN, int IV, int TX, int TY, int NY, int MINB>
__global__ void __launch_bounds__(TX* TY / NY, MINB)
    tbw_kernel(const __grid_constant__ KernelArgs<NS> args, const __grid_constant__ TwMaps maps, T* un2, int adjx,
               int kchunk) {
    using G = TwGeom<TX, TY, NY, T>;
    constexpr int UX = G::UX, IX = G::IX, IY = G::IY, D = G::D, NR = G::NR;
    constexpr unsigned SLOT = G::SLOT, SPLANE = G::SPLANE, ES = sizeof(T);
    using Mu = TwMem<T, UX, NY, IU, IUP, IV>;
    using Ms = TwMem<T, IX, NY, IU, IUP, IV>;
    extern __shared__ __align__(128) unsigned char tw_smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(tw_smem + D * SLOT + 5 * SPLANE);
    const unsigned rbase = smem_u32(tw_smem), sbase = rbase + D * SLOT;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int lo0 = args.lo[0], hi0 = args.hi[0], lo1 = args.lo[1], hi1 = args.hi[1], lo2 = args.lo[2],
              hi2 = args.hi[2];
    const int orgx = lo2 + blockIdx.x * TX, orgy = lo1 + blockIdx.y * TY;
    const int kb = lo0 + blockIdx.z * kchunk, ke = min(kb + kchunk, hi0);
    const int abase = kb - 4;                 // planes abase .. ke + 3 (TMA zero-fills outside the arrays)
    const int alast = ke + 3;

    // `un` (the step-1 output buffer and the boundary values of S1), un2 (step 2)
    T* unb = reinterpret_cast<T*>(args.arr[IUN].base);
    const long long n0 = args.arr[IUN].stride[0], n1 = args.arr[IUN].stride[1], n2 = args.arr[IUN].stride[2];
    // array extent (cells a boundary value may be read from): the nest pads by the stencil reach
    const int blo0 = lo0 - 2, bhi0 = hi0 + 2, blo1 = lo1 - 2, bhi1 = hi1 + 2, blo2 = lo2 - 2, bhi2 = hi2 + 2;

    // own cells (x, y + c): u-box / extended-tile byte offsets of cell 0
    const int x = orgx + tx, y = orgy + ty * NY;
    const unsigned ou = (unsigned)((ty * NY + 4) * UX + tx + 4) * ES;
    const unsigned oe = (unsigned)((ty * NY + 2) * IX + tx + 2) * ES;   // S1 plane
    const unsigned ov = (unsigned)((ty * NY + 2) * UX + tx + 4) * ES;   // up / vel2 boxes
    const long long go = (long long)y * n1 + (long long)x * n2;     // element offset of cell 0 in un / un2
    // halo-ring cell of the extended tile (threads 0..NR-1): rows 0, 1, IY-2, IY-1, then columns
    // 0, 1, IX-2, IX-1 interleaved (four lanes per row)
    int rex = 0, rey = 0;
    if (tid < 2 * IX) {
        rey = tid / IX;
        rex = tid - rey * IX;
    } else if (tid < 4 * IX) {
        rey = IY - 2 + (tid - 2 * IX) / IX;
        rex = (tid - 2 * IX) % IX;
    } else if (tid < NR) {
        const int j = tid - 4 * IX, side = j & 3;
        rex = side < 2 ? side : IX - 4 + side;
        rey = 2 + (j >> 2);
    }
    const bool has_ring = tid < NR;
    const int rx = orgx - 2 + rex, ry = orgy - 2 + rey;
    const unsigned ru = (unsigned)((rey + 2) * UX + rex + 2) * ES;
    const unsigned re = (unsigned)(rey * IX + rex) * ES;
    const unsigned rv = (unsigned)(rey * UX + rex + 2) * ES;
    const bool ring_xy_in = rx >= lo2 && rx < hi2 && ry >= lo1 && ry < hi1;
    const bool ring_xy_arr = rx >= blo2 && rx < bhi2 && ry >= blo1 && ry < bhi1;
    const long long rgo = (long long)ry * n1 + (long long)rx * n2;
    // hoisted per-cell predicates and plane pointers (one add per plane, no 64-bit multiplies)
    bool own_xy_in[NY], own_xy_arr[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) {
        own_xy_in[c] = x < hi2 && y + c < hi1;
        own_xy_arr[c] = x < bhi2 && y + c < bhi1;
    }
    T* unp = unb + (long long)(kb - 2) * n0 + go;       // own cell 0 at plane p (starts at kb - 2)
    T* rgp = unb + (long long)(kb - 2) * n0 + rgo;      // ring cell at plane p
    T* u2p = un2 + (long long)(kb - 4) * n0 + go;       // own cell 0 at plane q = p - 2

    auto issue = [&](int a, int s) {          // TMA of plane a (u, up, vel2 boxes) into slot s
        fence_proxy_async();
        mbar_expect_tx(&bars[s], (uint32_t)(G::UB + 2 * G::VB));
        unsigned char* d = tw_smem + s * SLOT;
        // every box starts at the u box's x origin: a TMA box whose inner start is not
        // 16-byte aligned faults (measured: illegal instruction), and orgx - 4 + adjx is
        const int cu[3] = {orgx - 4 + adjx, orgy - 4, a};
        const int cv[3] = {orgx - 4 + adjx, orgy - 2, a};
        tma_load<3>(d, &maps.u, cu, &bars[s]);
        tma_load<3>(d + G::OFF_UP, &maps.up, cv, &bars[s]);
        tma_load<3>(d + G::OFF_V, &maps.vel, cv, &bars[s]);
    };

    if (tid == 0) {
        tma_prefetch_desc(&maps.u);
        tma_prefetch_desc(&maps.up);
        tma_prefetch_desc(&maps.vel);
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < D && abase + s <= alast; ++s) issue(abase + s, s);

    // register queues (position of plane a: (a - abase) % 5; S1 of plane a: (a - kb + 2) % 5)
    T rq[NY][5], vq[NY][5], sq[NY][5], gq[5];
#pragma unroll
    for (int s = 0; s < 4; ++s) mbar_wait(&bars[s], 0);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int c = 0; c < NY; ++c) rq[c][s] = tb_lds(rbase + s * SLOT + ou + c * UX * ES, T(0));
        gq[s] = tb_lds(rbase + s * SLOT + ru, T(0));
    }
#pragma unroll
    for (int c = 0; c < NY; ++c)
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            vq[c][s] = sq[c][s] = T(0);
            if (s == 4) rq[c][s] = T(0);
        }
    gq[4] = T(0);
    __syncthreads();                          // slot 0 (plane abase) is free
    if (tid == 0 && abase + D <= alast) issue(abase + D, 0);

    int pt[3];
    uint32_t m = 0;                           // outer iteration: p0 = kb - 2 + 5 m
    for (int p0 = kb - 2; p0 <= ke + 1; p0 += 5, ++m) {
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int p = p0 + u;
            if (p > ke + 1) break;
            // plane p - abase = 5 m + 2 + u: slot(p) = (u + 2) % 5, slot(p + 2) = (u + 4) % 5,
            // slot(p - 1) = (u + 1) % 5 takes plane p + 4
            if (tid == 0 && p + 4 <= alast) issue(p + 4, (u + 1) % 5);
            mbar_wait(&bars[(u + 4) % 5], (m + (u + 4) / 5) & 1u);
            const unsigned sp = rbase + ((u + 2) % 5) * SLOT, sn = rbase + ((u + 4) % 5) * SLOT;
            const unsigned s1p = sbase + u * SPLANE;   // S1 ring slot of plane p
            const bool pin = p >= lo0 && p < hi0, parr = p >= blo0 && p < bhi0;
            const bool pstore = p >= kb && p < ke;
            // 1. step 1 on plane p: own cells, then the ring cell
#pragma unroll
            for (int c = 0; c < NY; ++c) rq[c][(u + 4) % 5] = tb_lds(sn + ou + c * UX * ES, T(0));
            T yc[NY];
#pragma unroll
            for (int c = 0; c < NY; ++c) yc[c] = rq[c][(u + 2) % 5];
#pragma unroll
            for (int c = 0; c < NY; ++c) {
                const T col[5] = {rq[c][u % 5], rq[c][(u + 1) % 5], rq[c][(u + 2) % 5], rq[c][(u + 3) % 5],
                                  rq[c][(u + 4) % 5]};
                const T upv = tb_lds(sp + G::OFF_UP + ov + c * UX * ES, T(0));
                const T vel = tb_lds(sp + G::OFF_V + ov + c * UX * ES, T(0));
                vq[c][(u + 2) % 5] = vel;
                T v = T(0);
                Mu mm{sp + ou + c * UX * ES, col, yc, c, upv, vel, &v};
                pt[0] = p;
                pt[1] = y + c;
                pt[2] = x;
                NS::template body<FORM>(mm, args.s, pt);
                const bool in = pin && own_xy_in[c];
                T s1 = v;
                if (!in) {                    // the un buffer's value: what step 2 would read there
                    s1 = T(0);
                    if (parr && own_xy_arr[c]) s1 = unp[c * n1];
                } else if (pstore) {
                    unp[c * n1] = v;
                }
                sq[c][u] = s1;
                tb_sts(s1p + oe + c * IX * ES, s1);
            }
            if (has_ring) {
                gq[(u + 4) % 5] = tb_lds(sn + ru, T(0));
                const T col[5] = {gq[u % 5], gq[(u + 1) % 5], gq[(u + 2) % 5], gq[(u + 3) % 5], gq[(u + 4) % 5]};
                const T upv = tb_lds(sp + G::OFF_UP + rv, T(0));
                const T vel = tb_lds(sp + G::OFF_V + rv, T(0));
                T v = T(0);
                Mu mm{sp + ru, col, col, -8, upv, vel, &v};   // c = -8: no register y-neighbours
                pt[0] = p;
                pt[1] = ry;
                pt[2] = rx;
                NS::template body<FORM>(mm, args.s, pt);
                T s1 = v;
                if (!(pin && ring_xy_in)) {
                    s1 = T(0);
                    if (parr && ring_xy_arr) s1 = *rgp;
                }
                tb_sts(s1p + re, s1);
            }
            __syncthreads();
            // 2. step 2 on plane q = p - 2: S1 column p-4 .. p, up = u(q), vel2(q)
            const int q = p - 2;
            if (q >= kb) {
                const unsigned s1q = sbase + ((u + 3) % 5) * SPLANE;
                T yq[NY];
#pragma unroll
                for (int c = 0; c < NY; ++c) yq[c] = sq[c][(u + 3) % 5];
#pragma unroll
                for (int c = 0; c < NY; ++c) {
                    const T col[5] = {sq[c][(u + 1) % 5], sq[c][(u + 2) % 5], sq[c][(u + 3) % 5], sq[c][(u + 4) % 5],
                                      sq[c][u % 5]};
                    T v = T(0);
                    Ms mm{s1q + oe + c * IX * ES, col, yq, c, rq[c][u % 5], vq[c][u % 5], &v};
                    pt[0] = q;
                    pt[1] = y + c;
                    pt[2] = x;
                    NS::template body<FORM>(mm, args.s, pt);
                    if (own_xy_in[c]) u2p[c * n1] = v;
                }
            }
            unp += n0;
            rgp += n0;
            u2p += n0;
        }
    }
}

template <class NS, class T, int IU, int IUP, int IV, int TX, int TY, int NY>
bool encode_tw_maps(const LaunchReq& r, TwMaps& maps, int& adjx) {
    using G = TwGeom<TX, TY, NY, T>;
    EncodeTiledFn enc = tma_encoder();
    if (!enc) return false;
    const int want[3] = {IU, IUP, IV};
    CUtensorMap* out[3] = {&maps.u, &maps.up, &maps.vel};
    for (int w = 0; w < 3; ++w) {
        const acs_array* d = nullptr;
        for (int i = 0; i < r.n_arrays; ++i)
            if (r.arrays[i].name && std::strcmp(r.arrays[i].name, NS::array_names[want[w]]) == 0) d = &r.arrays[i];
        if (!d || d->ndim != 3) return false;
        long long st[3];
        bool rm = true;
        for (int p = 0; p < 3; ++p) rm = rm && d->strides[p] == 0;
        st[2] = rm ? 1 : d->strides[2];
        st[1] = rm ? d->dims[2] : d->strides[1];
        st[0] = rm ? d->dims[1] * d->dims[2] : d->strides[0];
        const int es = (int)sizeof(T);
        const int mis = (int)(reinterpret_cast<uintptr_t>(d->data) % 16);
        if (st[2] != 1 || mis % es != 0 || (st[1] * es) % 16 != 0 || (st[0] * es) % 16 != 0 || st[0] < st[1])
            return false;
        const int adj = mis / es;
        if (w == 0) adjx = adj;
        else if (adj != adjx) return false;   // one x shift for every box
        cuuint64_t gdim[3] = {(cuuint64_t)(d->dims[2] + adj), (cuuint64_t)d->dims[1], (cuuint64_t)d->dims[0]};
        cuuint64_t gstr[2] = {(cuuint64_t)(st[1] * es), (cuuint64_t)(st[0] * es)};
        cuuint32_t box[3] = {(cuuint32_t)G::UX, (cuuint32_t)(w == 0 ? G::UY : G::IY), 1u};
        cuuint32_t estr[3] = {1u, 1u, 1u};
        void* base = static_cast<char*>(d->data) - (size_t)adj * es;
        const CUtensorMapDataType dt =
            sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        if (enc(out[w], dt, 3u, base, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

// two leapfrog steps per launch; the request carries the nest's arrays plus
// "un2" (the fourth buffer, un's shape and strides)
template <class NS, class T, int FORM, int IU, int IUP, int IUN, int IV, int TX, int TY, int NY, int MINB>
acs_status launch_tbw(const LaunchReq& r) {
    static_assert(TwPlan<NS, IU, IUP, IUN, IV>::usable(), "tbw: not a 3-level leapfrog star stencil of radius 2");
    using G = TwGeom<TX, TY, NY, T>;
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    if (r.shard) {
        set_error("tbw: two-step launches are not sharded");
        return ACS_E_ARG;
    }
    const acs_array *un = nullptr, *un2 = nullptr;
    for (int i = 0; i < r.n_arrays; ++i) {
        if (r.arrays[i].name && std::strcmp(r.arrays[i].name, NS::array_names[IUN]) == 0) un = &r.arrays[i];
        if (r.arrays[i].name && std::strcmp(r.arrays[i].name, "un2") == 0) un2 = &r.arrays[i];
    }
    if (!un || !un2 || !un2->data || un2->ndim != un->ndim || un2->dtype != un->dtype) {
        set_error("tbw: a fourth buffer 'un2' of un's shape and dtype is required");
        return ACS_E_ARG;
    }
    for (int p = 0; p < un->ndim; ++p)
        if (un2->dims[p] != un->dims[p] || un2->strides[p] != un->strides[p] ||
            (reinterpret_cast<uintptr_t>(un2->data) - reinterpret_cast<uintptr_t>(un->data)) % 16 != 0) {
            set_error("tbw: 'un2' must have un's dims, strides and 16-byte phase");
            return ACS_E_SHAPE;
        }
    auto kern = tbw_kernel<NS, T, FORM, IU, IUP, IUN, IV, TX, TY, NY, MINB>;
    if (r.preload) return preload_fn((const void*)kern);
    TwMaps maps;
    int adjx = 0;
    if (!encode_tw_maps<NS, T, IU, IUP, IV, TX, TY, NY>(r, maps, adjx)) {
        set_error("tbw: the TMA cannot describe this layout (16-byte aligned pitches, one x phase); use native strides");
        return ACS_E_LAYOUT;
    }
    static std::atomic<unsigned long long> attr_done{0};
    set_smem_attr_once(kern, G::smem, attr_done);
    const long long nx = ka.hi[2] - ka.lo[2], ny = ka.hi[1] - ka.lo[1], nz = ka.hi[0] - ka.lo[0];
    const long long tiles = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
    // 96-plane chunks (measured best of 64 / 80 / 96 / 128 / 192 / 256 at 1024^3,
    // profiles/r02_wave4_tb2.md); never below 24 (6 extra planes per chunk)
    long long kchunk = 96;
    (void)tiles;
    static const long long kch_env = [] {   // experiment knob (tools/gpu), not a tuning path
        const char* e = std::getenv("ACS_TB_KCHUNK");
        return e ? std::atoll(e) : 0LL;
    }();
    if (kch_env > 0) kchunk = kch_env;
    if (kchunk < 24) kchunk = 24;
    if (kchunk > nz) kchunk = nz;
    const long long chunks = (nz + kchunk - 1) / kchunk;
    dim3 grid((unsigned)((nx + TX - 1) / TX), (unsigned)((ny + TY - 1) / TY), (unsigned)chunks);
    kern<<<grid, dim3(TX, TY / NY, 1), G::smem, r.stream>>>(ka, maps, static_cast<T*>(un2->data), adjx, (int)kchunk);
    return check_launch("tbw");
}

template <class NS, class T, int IU, int IUP, int IUN, int IV, int TX, int TY, int NY, int MINB>
void fill_tbw(Entry& e, int prec) {
    e.tb2[prec][0] = &launch_tbw<NS, T, 0, IU, IUP, IUN, IV, TX, TY, NY, MINB>;
    e.tb2[prec][1] = &launch_tbw<NS, T, 1, IU, IUP, IUN, IV, TX, TY, NY, MINB>;
    e.tb2[prec][2] = &launch_tbw<NS, T, 2, IU, IUP, IUN, IV, TX, TY, NY, MINB>;
    e.tb2[prec][3] = &launch_tbw<NS, T, 3, IU, IUP, IUN, IV, TX, TY, NY, MINB>;
    e.tb2[prec][4] = &launch_tbw<NS, T, 4, IU, IUP, IUN, IV, TX, TY, NY, MINB>;
    e.tb2_name[prec] = "temporal block x2, leapfrog (TMA ring of u/up/vel2 boxes, register columns, 4th buffer), tile " +
                       std::to_string(TX) + "x" + std::to_string(TY) + ", " + std::to_string(NY) + " y-cells per thread";
    e.tb2_read = IU;
}

}  // namespace acs
