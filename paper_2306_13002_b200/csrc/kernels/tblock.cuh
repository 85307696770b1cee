// tblock.cuh — temporal blocking: two time steps of a ping-pong star stencil
// per launch (Jacobi-7).
//
// A ping-pong nest (one array R read with a radius-1 star stencil, one array
// W written at the point; the time loop swaps the two) advances by two steps
// in one pass over HBM.  A CTA of TX x TY threads owns a TX x TY output tile
// and marches along k over a chunk of planes; per march plane p:
//   0. one elected thread refills the R ring: a cp.async.bulk.tensor (TMA)
//      box of (TX+4) x (TY+4) cells (2-cell halo) per plane into a 6-plane
//      ring (PF = 4 planes ahead), completion on the slot's mbarrier;
//   1. step 1 on the EXTENDED tile (TX+2) x (TY+2) of plane p: every thread
//      its own cell, threads 0..NR-1 also one cell of the halo ring.  The
//      cell's own column (k-1, k, k+1) lives in a register queue (one LDS of
//      the new top plane per step), the four in-plane neighbours are LDS at
//      compile-time offsets.  The step-1 field goes to a 3-plane shared ring
//      — it never reaches HBM;
//   2. (after the one barrier per plane) step 2 on the tile of plane p-1:
//      the column again from a register queue of the thread's own step-1
//      values, the in-plane neighbours from the step-1 ring; one STG to W.
// The plane loop is unrolled by 6, so the ring slots, both queues and the
// step-1 ring slot are compile-time (queue shifts are register renames).
//
// HBM traffic per two steps: R read once, W written once — 16 B/point for two
// steps of an f64 nest instead of 32 (the bench reports the algorithmic bytes
// of the two steps and the DRAM bytes ncu measures, separately).  The step-1
// field outside the iteration space (the nest's fixed boundary) is R's value
// there: both buffers of the ping-pong must carry the same boundary (true for
// the nest's time loop, whose boundary is never written).  The same generated
// body as every other skeleton, so results are bit-identical to two launches
// of the single-step kernel (tests/test_gpu_parity.py).
#pragma once

#include <cstdlib>

#include "../acs_device.cuh"
#include "../registry.hpp"
#include "../tma.cuh"

namespace acs {

template <class NS>
struct TbPlan {
    static constexpr int R = NS::NARR == 2 && NS::readonly(0) ? 0 : 1;   // the array read
    static constexpr int W = 1 - R;                                      // the array written
    static constexpr bool usable() {
        if (NS::NARR != 2 || NS::NLOOP != 3 || NS::has_dynamic_index) return false;
        if (!NS::readonly(R) || NS::readonly(W) || NS::is_loaded(W) || NS::is_int(R) || NS::is_int(W)) return false;
        for (int p = 0; p < 3; ++p) {
            if (NS::ld_sig(R, p) != p || NS::ld_lo(R, p) < -1 || NS::ld_hi(R, p) > 1) return false;
            if (NS::sig(W, p) != p || NS::sig(R, p) != p) return false;
        }
        if (NS::NSROW != 1 || NS::srow_arr(0) != W) return false;
        for (int p = 0; p < 3; ++p)
            if (NS::srow_off(0, p) != 0) return false;
        // a star: rows off the march plane are single centre cells (the register queue)
        for (int r = 0; r < NS::NROW; ++r)
            if (NS::row_off(r, 0) != 0 && (NS::row_off(r, 1) != 0 || NS::row_xlo(r) != 0 || NS::row_xhi(r) != 0))
                return false;
        return true;
    }
};

// shared-window (32-bit) loads / stores: the addresses stay plain integers, so
// the loop-invariant parts are computed once per thread, not per access
__device__ __forceinline__ double tb_lds(unsigned a, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float tb_lds(unsigned a, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void tb_sts(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ void tb_sts(unsigned a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }

// memory policy of one point: the column (k-1, k, k+1) from registers, the
// y neighbours from registers when the thread owns them too, the other
// in-plane neighbours from shared memory at `a` (this cell's byte address in
// the current plane, row stride RS elements); the store lands in *out
template <class T, int RS>
struct TbMem {
    unsigned a;
    T qm, q0, qp;
    T ym, yp;      // in-plane y-1 / y+1 neighbours held by this thread (its other cells), if hym / hyp
    bool hym, hyp; // compile-time constants once the cell loop is unrolled
    T* out;
    T xm = T(0), xp = T(0);          // x-1 / x+1 from the adjacent lanes (warp shuffle), if hx;
    bool hx = false, l0 = false, l31 = false;   // lanes 0 / 31 (the tile edge) read shared memory
    template <int ARR>
    using elem_t = T;
    template <int ARR, int... O>
    __device__ __forceinline__ T ld() const {
        constexpr int off[sizeof...(O)] = {O...};
        if constexpr (off[1] == 0 && off[2] == 0) {
            return off[0] < 0 ? qm : (off[0] > 0 ? qp : q0);
        } else {
            static_assert(off[0] == 0, "tb2: off-plane loads are centre cells (a star stencil)");
            if constexpr (off[1] == -1 && off[2] == 0)
                if (hym) return ym;
            if constexpr (off[1] == 1 && off[2] == 0)
                if (hyp) return yp;
            if constexpr (off[1] == 0 && (off[2] == 1 || off[2] == -1))
                if (hx) {
                    constexpr int cx = off[2] * (int)sizeof(T);
                    T v = off[2] < 0 ? xm : xp;
                    if (off[2] < 0 ? l0 : l31) v = tb_lds(a + (unsigned)cx, T(0));
                    return v;
                }
            constexpr int c = (off[1] * RS + off[2]) * (int)sizeof(T);
            return tb_lds(a + (unsigned)c, T(0));
        }
    }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(T v) const {
        *out = v;
    }
    template <int ARR, class... I>
    __device__ __forceinline__ T ldx(I...) const { return T(0); }       // not reached: no dynamic index
    template <int ARR, class... I>
    __device__ __forceinline__ T ldx_in(I...) const { return T(0); }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A...) const {}
};

template <int TX, int TY, int NY, int PF, class T>
struct TbGeom {
    static constexpr int EX = TX + 4, EY = TY + 4;     // staged R box (2-cell halo)
    static constexpr int IX = TX + 2, IY = TY + 2;     // step-1 plane (extended tile)
    static constexpr int D = 6;                        // R ring planes (PF = 4 in flight)
    static constexpr int NT = TX * TY / NY;           // threads: NY cells of a column each
    static constexpr int NR = IX * IY - TX * TY;       // halo-ring cells of the extended tile
    static constexpr unsigned PLANE = ((EY * EX * (int)sizeof(T) + 127) / 128) * 128;
    static constexpr unsigned IPLANE = ((IY * IX * (int)sizeof(T) + 127) / 128) * 128;
    static constexpr int smem = D * PLANE + 3 * IPLANE + D * 8;
    static_assert(PF == D - 2, "tb2: the ring is 6 planes deep (PF = 4)");
    static_assert(NR <= NT, "tb2: the halo ring needs at most one cell per thread");
    static_assert(TY % NY == 0, "tb2: NY divides the tile height");
    static_assert((EX * (int)sizeof(T)) % 16 == 0, "tb2: TMA box rows are 16-byte multiples");
};

template <class NS, class T, int FORM, int TX, int TY, int NY, int PF, int MINB, int XS>
__global__ void __launch_bounds__(TX* TY / NY, MINB) tb2_kernel(const __grid_constant__ KernelArgs<NS> args,
                                                             const __grid_constant__ CUtensorMap rmap, int adjx,
                                                             int kchunk) {
    using G = TbGeom<TX, TY, NY, PF, T>;
    constexpr int R = TbPlan<NS>::R, W = TbPlan<NS>::W;
    constexpr int EX = G::EX, IX = G::IX, IY = G::IY, D = G::D, NR = G::NR;
    constexpr unsigned PLANE = G::PLANE, IPLANE = G::IPLANE, ES = sizeof(T);
    extern __shared__ __align__(128) unsigned char tb_smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(tb_smem + D * PLANE + 3 * IPLANE);
    const unsigned rbase = smem_u32(tb_smem), ibase = rbase + D * PLANE;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int lo0 = args.lo[0], hi0 = args.hi[0], lo1 = args.lo[1], hi1 = args.hi[1], lo2 = args.lo[2],
              hi2 = args.hi[2];
    const int orgx = lo2 + blockIdx.x * TX, orgy = lo1 + blockIdx.y * TY;
    const int kb = lo0 + blockIdx.z * kchunk, ke = min(kb + kchunk, hi0);
    const int abase = kb - 2;                 // R planes abase .. ke + 1 (TMA zero-fills outside the array)
    const int alast = ke + 1;

    // own cells (x, y + c), c < NY: box / step-1-plane byte offsets of cell 0, domain flags, W offset
    const int x = orgx + tx, y = orgy + ty * NY;
    const unsigned obox = (unsigned)((ty * NY + 2) * EX + tx + 2) * ES;
    const unsigned oint = (unsigned)((ty * NY + 1) * IX + tx + 1) * ES;
    bool own_in[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) own_in[c] = x < hi2 && y + c < hi1;
    T* wp = reinterpret_cast<T*>(args.arr[W].base) + (long long)y * args.arr[W].stride[1] +
            (long long)x * args.arr[W].stride[2];
    const long long w0 = args.arr[W].stride[0], w1 = args.arr[W].stride[1];
    // halo-ring cell (threads 0..NR-1): top row, bottom row, then the left and right columns
    // interleaved (lane pairs share a row: half the bank conflicts of a column walk)
    int rex = 0, rey = 0;
    if (tid < IX) {
        rex = tid;
        rey = 0;
    } else if (tid < 2 * IX) {
        rex = tid - IX;
        rey = IY - 1;
    } else if (tid < NR) {
        rex = ((tid - 2 * IX) & 1) ? IX - 1 : 0;
        rey = ((tid - 2 * IX) >> 1) + 1;
    }                                         // other threads: cell (0, 0), in the box (never stored)
    const bool has_ring = tid < NR;
    const int rx = orgx - 1 + rex, ry = orgy - 1 + rey;
    const bool ring_in = rx >= lo2 && rx < hi2 && ry >= lo1 && ry < hi1;
    const unsigned rbox = (unsigned)((rey + 1) * EX + rex + 1) * ES;
    const unsigned rint = (unsigned)(rey * IX + rex) * ES;

    // R plane a lives in ring slot (a - abase) % D, its fill number (a - abase) / D
    auto issue = [&](int a, int s) {          // TMA of R plane a into slot s (elected thread)
        fence_proxy_async();
        mbar_expect_tx(&bars[s], (uint32_t)(G::EY * EX * ES));
        const int c[3] = {orgx - 2 + adjx, orgy - 2, a};
        tma_load<3>(tb_smem + s * PLANE, &rmap, c, &bars[s]);
    };

    if (tid == 0) {
        tma_prefetch_desc(&rmap);
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < D && abase + s <= alast; ++s) issue(abase + s, s);

    // register queues: R column of the own / ring cells, step-1 column of the own cells
    T rq[NY][3], gq[3], sq[NY][3];
    mbar_wait(&bars[0], 0);
    mbar_wait(&bars[1], 0);
#pragma unroll
    for (int c = 0; c < NY; ++c) {
        rq[c][0] = tb_lds(rbase + obox + c * EX * ES, T(0));
        rq[c][1] = tb_lds(rbase + PLANE + obox + c * EX * ES, T(0));
        rq[c][2] = sq[c][0] = sq[c][1] = sq[c][2] = T(0);
    }
    gq[0] = tb_lds(rbase + rbox, T(0));
    gq[1] = tb_lds(rbase + PLANE + rbox, T(0));
    gq[2] = T(0);
    __syncthreads();                          // plane abase's slot is free for the refill

    int pt[3];
    // the plane loop, unrolled by D = 6: plane p = p0 + u has R slot (u + 1) % 6,
    // step-1 slot u % 3 and queue positions u % 3 .. (u + 2) % 3 — all compile-time
    uint32_t fill = 0;                        // (p0 - kb + 1) / 6: fill number of slot 1.. at phase 0
    for (int p0 = kb - 1; p0 <= ke; p0 += D, ++fill) {
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const int p = p0 + u;
            if (p > ke) break;
            // queue slots of this phase: plane p-1, p, p+1 = (u), (u+1), (u+2) mod 3 (R queues);
            // step-1 values of planes p-2, p-1, p likewise (sq)
            const int qm = u % 3, qc = (u + 1) % 3, qn = (u + 2) % 3;
            const int sl_p = (u + 1) % D, sl_n = (u + 2) % D, sl_free = u % D;
            // slot u held plane p - 1 (read by the previous phase, before its barrier)
            if (tid == 0 && p - 1 + D <= alast) issue(p - 1 + D, sl_free);
            mbar_wait(&bars[sl_n], (fill + (u + 2) / D) & 1u);
            const unsigned sp = rbase + sl_p * PLANE, sn = rbase + sl_n * PLANE;
            const unsigned ip = ibase + (unsigned)(u % 3) * IPLANE;    // step-1 slot of plane p
            const bool pin = p >= lo0 && p < hi0;
            // 1. step 1 on plane p: own cells, then the ring cell
#pragma unroll
            for (int c = 0; c < NY; ++c) rq[c][qn] = tb_lds(sn + obox + c * EX * ES, T(0));
#pragma unroll
            for (int c = 0; c < NY; ++c) {
                T v = T(0);
                TbMem<T, EX> m{sp + obox + c * EX * ES, rq[c][qm], rq[c][qc], rq[c][qn], rq[c > 0 ? c - 1 : 0][qc],
                               rq[c < NY - 1 ? c + 1 : 0][qc], c > 0, c < NY - 1, &v};
                if constexpr (XS) {           // x neighbours from the adjacent lanes (a warp is one row)
                    m.xm = __shfl_up_sync(0xffffffffu, rq[c][qc], 1);
                    m.xp = __shfl_down_sync(0xffffffffu, rq[c][qc], 1);
                    m.hx = true;
                    m.l0 = tx == 0;
                    m.l31 = tx == 31;
                }
                pt[0] = p;
                pt[1] = y + c;
                pt[2] = x;
                NS::template body<FORM>(m, args.s, pt);
                const T s1 = pin && own_in[c] ? v : rq[c][qc];
                sq[c][qn] = s1;
                tb_sts(ip + oint + c * IX * ES, s1);
            }
            if (has_ring) {
                gq[qn] = tb_lds(sn + rbox, T(0));
                T v = T(0);
                TbMem<T, EX> m{sp + rbox, gq[qm], gq[qc], gq[qn], T(0), T(0), false, false, &v};
                pt[0] = p;
                pt[1] = ry;
                pt[2] = rx;
                NS::template body<FORM>(m, args.s, pt);
                tb_sts(ip + rint, pin && ring_in ? v : gq[qc]);
            }
            __syncthreads();
            // 2. step 2 on plane q = p - 1 (its step-1 slot is u - 1 mod 3)
            const int q = p - 1;
            if (q >= kb) {
                const unsigned iq = ibase + (unsigned)((u + 2) % 3) * IPLANE;   // plane p - 1
#pragma unroll
                for (int c = 0; c < NY; ++c) {
                    T v = T(0);
                    // the own step-1 column of planes q-1, q, q+1 = p-2, p-1, p
                    TbMem<T, IX> m{iq + oint + c * IX * ES, sq[c][qm], sq[c][qc], sq[c][qn], sq[c > 0 ? c - 1 : 0][qc],
                                   sq[c < NY - 1 ? c + 1 : 0][qc], c > 0, c < NY - 1, &v};
                    if constexpr (XS) {
                        m.xm = __shfl_up_sync(0xffffffffu, sq[c][qc], 1);
                        m.xp = __shfl_down_sync(0xffffffffu, sq[c][qc], 1);
                        m.hx = true;
                        m.l0 = tx == 0;
                        m.l31 = tx == 31;
                    }
                    pt[0] = q;
                    pt[1] = y + c;
                    pt[2] = x;
                    NS::template body<FORM>(m, args.s, pt);
                    if (own_in[c]) wp[(long long)q * w0 + c * w1] = v;
                }
            }
        }
    }
}

template <class NS, class T, int TX, int TY, int NY, int PF>
bool encode_tb_map(const LaunchReq& r, CUtensorMap& map, int& adjx) {
    constexpr int R = TbPlan<NS>::R;
    using G = TbGeom<TX, TY, NY, PF, T>;
    EncodeTiledFn enc = tma_encoder();
    if (!enc) return false;
    const acs_array* d = nullptr;
    for (int i = 0; i < r.n_arrays; ++i)
        if (std::strcmp(r.arrays[i].name, NS::array_names[R]) == 0) d = &r.arrays[i];
    if (!d || d->ndim != 3) return false;
    long long st[3];
    bool rm = true;
    for (int p = 0; p < 3; ++p) rm = rm && d->strides[p] == 0;
    st[2] = rm ? 1 : d->strides[2];
    st[1] = rm ? d->dims[2] : d->strides[1];
    st[0] = rm ? d->dims[1] * d->dims[2] : d->strides[0];
    const int es = (int)sizeof(T);
    const int mis = (int)(reinterpret_cast<uintptr_t>(d->data) % 16);
    if (st[2] != 1 || mis % es != 0 || (st[1] * es) % 16 != 0 || (st[0] * es) % 16 != 0 || st[0] < st[1]) return false;
    adjx = mis / es;
    cuuint64_t gdim[3] = {(cuuint64_t)(d->dims[2] + adjx), (cuuint64_t)d->dims[1], (cuuint64_t)d->dims[0]};
    cuuint64_t gstr[2] = {(cuuint64_t)(st[1] * es), (cuuint64_t)(st[0] * es)};
    cuuint32_t box[3] = {(cuuint32_t)G::EX, (cuuint32_t)G::EY, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    void* base = static_cast<char*>(d->data) - (size_t)adjx * es;
    const CUtensorMapDataType dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    return enc(&map, dt, 3u, base, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class NS, class T, int FORM, int TX, int TY, int NY, int PF, int MINB, int XS = 0>
acs_status launch_tb2(const LaunchReq& r) {
    static_assert(!XS || TX == 32, "tb2: the x-shuffle needs one warp per tile row");
    static_assert(TbPlan<NS>::usable(), "tb2: not a ping-pong star stencil");
    using G = TbGeom<TX, TY, NY, PF, T>;
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    if (r.shard) {
        set_error("tb2: two-step launches are not sharded");
        return ACS_E_ARG;
    }
    auto kern = tb2_kernel<NS, T, FORM, TX, TY, NY, PF, MINB, XS>;
    if (r.preload) return preload_fn((const void*)kern);
    CUtensorMap map;
    int adjx = 0;
    if (!encode_tb_map<NS, T, TX, TY, NY, PF>(r, map, adjx)) {
        set_error(std::string("tb2 (") + NS::array_names[TbPlan<NS>::R] +
                  "): the TMA cannot describe this layout (16-byte aligned pitches needed); use native strides");
        return ACS_E_LAYOUT;
    }
    static std::atomic<unsigned long long> attr_done{0};
    set_smem_attr_once(kern, G::smem, attr_done);
    const long long nx = ka.hi[2] - ka.lo[2], ny = ka.hi[1] - ka.lo[1], nz = ka.hi[0] - ka.lo[0];
    const long long tiles = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
    // ~4 waves of the resident CTAs; chunks long enough to amortise the 3 extra planes
    long long kchunk = (nz * tiles + 148LL * 4 * MINB - 1) / (148LL * 4 * MINB);
    static const long long kch_env = [] {   // experiment knob (tools/gpu), not a tuning path
        const char* e = std::getenv("ACS_TB_KCHUNK");
        return e ? std::atoll(e) : 0LL;
    }();
    if (kch_env > 0) kchunk = kch_env;
    if (kchunk < 12) kchunk = 12;
    if (kchunk > nz) kchunk = nz;
    const long long chunks = (nz + kchunk - 1) / kchunk;
    dim3 grid((unsigned)((nx + TX - 1) / TX), (unsigned)((ny + TY - 1) / TY), (unsigned)chunks);
    kern<<<grid, dim3(TX, TY / NY, 1), G::smem, r.stream>>>(ka, map, adjx, (int)kchunk);
    return check_launch("tb2");
}

// the registered two-step schedules of a nest: configuration 0 is the default;
// ACS_TB_CFG=<i> picks another one (an experiment knob for tools/gpu, not a tuning path)
template <int TX, int TY, int NY, int PF, int MINB, int XS = 0>
struct TbCfg {};

template <class NS, class T, int FORM, int... A>
acs_status launch_tb2_cfg(const LaunchReq& r, TbCfg<A...>) {
    return launch_tb2<NS, T, FORM, A...>(r);
}

inline int tb_cfg_env() {
    static const int v = [] {
        const char* e = std::getenv("ACS_TB_CFG");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

template <class NS, class T, int FORM, class C0, class... Cs>
acs_status launch_tb2_set(const LaunchReq& r) {
    const int want = tb_cfg_env();
    int i = 0;
    acs_status st = ACS_E_ARG;
    bool done = false;
    auto one = [&](auto cfg) {
        if (!done && i++ == want) {
            st = launch_tb2_cfg<NS, T, FORM>(r, cfg);
            done = true;
        }
    };
    one(C0{});
    (one(Cs{}), ...);
    if (!done) st = launch_tb2_cfg<NS, T, FORM>(r, C0{});
    return st;
}

template <int TX, int TY, int NY, int PF, int MINB, int XS>
std::string tb2_name_of(TbCfg<TX, TY, NY, PF, MINB, XS>) {
    return "temporal block x2 (TMA ring, register columns), tile " + std::to_string(TX) + "x" + std::to_string(TY) +
           ", " + std::to_string(NY) + " y-cell(s) per thread, pf " + std::to_string(PF) +
           (XS ? ", x neighbours by warp shuffle" : "");
}

template <class NS, class T, class C0, class... Cs>
void fill_tb2(Entry& e, int prec) {
    e.tb2[prec][0] = &launch_tb2_set<NS, T, 0, C0, Cs...>;
    e.tb2[prec][1] = &launch_tb2_set<NS, T, 1, C0, Cs...>;
    e.tb2[prec][2] = &launch_tb2_set<NS, T, 2, C0, Cs...>;
    e.tb2[prec][3] = &launch_tb2_set<NS, T, 3, C0, Cs...>;
    e.tb2[prec][4] = &launch_tb2_set<NS, T, 4, C0, Cs...>;
    e.tb2_name[prec] = [](auto c) { return tb2_name_of(c); }(C0{});
    e.tb2_read = TbPlan<NS>::R;
}

}  // namespace acs
