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

// ---- register queue along the march -----------------------------------------
// For slice S of form FORM, every read-only array field the slice loads at
// offsets only along the outermost loop (zsolve: fjacZ[m][n][k-1..k+1],
// njacZ[m][n][k-1..k+1]) is kept as a queue of its k-offset range in
// registers: per step one LDG of the newest plane, the rest shifted from the
// previous step (the paper's common loads held in registers, across
// iterations of the marched loop).
struct QField {
    int arr = -1;
    int ref = -1;            // a representative sl_off row (other positions' offsets)
    int dzlo = 0, dzhi = 0;
    int qoff = 0;
};

template <int MAXF>
struct QTable {
    QField f[MAXF];
    int n = 0;
    int total = 0;
};

template <class NS, int FORM, int S>
struct QPlan {
    static constexpr int MAXF = 64;
    static constexpr int mpos(int a) {
        for (int p = 0; p < NS::ndim(a); ++p)
            if (NS::sig(a, p) == 0) return p;
        return -1;
    }
    static constexpr bool eligible(int i) {
        if constexpr (FORM == 0) {
            return false;
        } else {
            const int a = NS::sl_arr(i), mp = mpos(a);
            if (mp < 0 || !NS::readonly(a) || NS::is_int(a)) return false;
            for (int p = 0; p < NS::ndim(a); ++p)
                if (NS::sig(a, p) > 0 && NS::sl_off(i, p) != 0) return false;
            return true;
        }
    }
    static constexpr bool same_field(int i, int j) {
        const int a = NS::sl_arr(i);
        if (NS::sl_arr(j) != a) return false;
        for (int p = 0; p < NS::ndim(a); ++p)
            if (p != mpos(a) && NS::sl_off(i, p) != NS::sl_off(j, p)) return false;
        return true;
    }
    static constexpr QTable<MAXF> build() {
        QTable<MAXF> t{};
        if (S >= NS::nslices[FORM]) return t;
        const int b = NS::sl_first(FORM, S), n = NS::sl_nref(FORM, S);
        for (int i = b; i < b + n; ++i) {
            if (!eligible(i)) continue;
            const int dz = NS::sl_off(i, mpos(NS::sl_arr(i)));
            int k = -1;
            for (int j = 0; j < t.n && k < 0; ++j)
                if (same_field(t.f[j].ref, i)) k = j;
            if (k < 0) {
                if (t.n >= MAXF) return QTable<MAXF>{};
                k = t.n++;
                t.f[k].arr = NS::sl_arr(i);
                t.f[k].ref = i;
                t.f[k].dzlo = t.f[k].dzhi = dz;
            } else {
                if (dz < t.f[k].dzlo) t.f[k].dzlo = dz;
                if (dz > t.f[k].dzhi) t.f[k].dzhi = dz;
            }
        }
        for (int k = 0; k < t.n; ++k) {
            t.f[k].qoff = t.total;
            t.total += t.f[k].dzhi - t.f[k].dzlo + 1;
        }
        return t;
    }
    static constexpr QTable<MAXF> Q = build();
    static constexpr int total() { return Q.total > 0 ? Q.total : 1; }
    template <int ARR, int... O>
    static constexpr int field_of() {
        constexpr int off[sizeof...(O)] = {O...};
        for (int k = 0; k < Q.n; ++k) {
            if (Q.f[k].arr != ARR) continue;
            bool ok = true;
            for (int p = 0; p < (int)sizeof...(O); ++p)
                if (p != mpos(ARR) && NS::sl_off(Q.f[k].ref, p) != off[p]) ok = false;
            if (ok && off[mpos(ARR)] >= Q.f[k].dzlo && off[mpos(ARR)] <= Q.f[k].dzhi) return k;
        }
        return -1;
    }
    // element offset of field K at march offset DZ relative to the point
    template <int K, int DZ, class G, int... PP>
    static __device__ __forceinline__ long long index(const G& g, std::integer_sequence<int, PP...>) {
        constexpr int A = Q.f[K].arr, R = Q.f[K].ref, MP = mpos(A);
        return g.template static_index<A, (PP == MP ? DZ : NS::sl_off(R, PP))...>();
    }
};

template <class NS, class T, int FORM, int S>
struct QMem {
    using QP = QPlan<NS, FORM, S>;
    NaiveMem<NS, T, FORM == ACS_ORIGINAL> g;
    const T* q;
    template <int ARR>
    using elem_t = typename NaiveMem<NS, T, FORM == ACS_ORIGINAL>::template elem_t<ARR>;
    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const {
        constexpr int k = QP::template field_of<ARR, O...>();
        if constexpr (k >= 0) {
            constexpr int off[sizeof...(O)] = {O...};
            constexpr int idx = QP::Q.f[k].qoff + off[QP::mpos(ARR)] - QP::Q.f[k].dzlo;
            return q[idx];
        } else {
            return g.template ld<ARR, O...>();
        }
    }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... ii) const { return g.template ldx<ARR>(ii...); }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx_in(I... ii) const { return g.template ldx<ARR>(ii...); }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const { g.template st<ARR, O...>(v); }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const { g.template stx<ARR>(args...); }
};

// fill queue field K at march offsets [DZ, dzhi]
template <class NS, class QP, class G, class T, int K, int DZ>
__device__ __forceinline__ void q_fill(const G& g, T* q) {
    if constexpr (DZ <= QP::Q.f[K].dzhi) {
        constexpr int A = QP::Q.f[K].arr;
        constexpr int slot = QP::Q.f[K].qoff + DZ - QP::Q.f[K].dzlo;
        const long long idx = QP::template index<K, DZ>(g, std::make_integer_sequence<int, NS::ndim(A)>{});
        q[slot] = g.template load_at<A>(idx);
        q_fill<NS, QP, G, T, K, DZ + 1>(g, q);
    }
}

// one march step of every queue: all offsets on the chunk's first plane,
// afterwards shift by one plane and load only the newest
template <class NS, class QP, class G, class T, int K>
__device__ __forceinline__ void q_step(const G& g, T* q, bool first) {
    if constexpr (K < QP::Q.n) {
        constexpr int lo = QP::Q.f[K].dzlo, hi = QP::Q.f[K].dzhi, base = QP::Q.f[K].qoff;
        if (first) {
            q_fill<NS, QP, G, T, K, lo>(g, q);
        } else {
#pragma unroll
            for (int i = 0; i < hi - lo; ++i) q[base + i] = q[base + i + 1];
            q_fill<NS, QP, G, T, K, hi>(g, q);
        }
        q_step<NS, QP, G, T, K + 1>(g, q, first);
    }
}

// the k march of one slice, the slice a compile-time constant: no switch in
// the loop, so the loads of several planes can be issued ahead (unroll)
template <class NS, class T, int FORM, int S, int UNR>
__device__ __forceinline__ void march_slice(NaiveMem<NS, T, FORM == ACS_ORIGINAL>& m, const KernelArgs<NS>& args,
                                            int* pt, int slice, int kb, int ke) {
    if constexpr (S < NS::nslices[FORM]) {
        if (slice == S) {
            using QP = QPlan<NS, FORM, S>;
            using G = NaiveMem<NS, T, FORM == ACS_ORIGINAL>;
            if constexpr (QP::Q.n > 0) {
                T q[QP::total()];
                if (kb < ke) {   // first plane of the chunk: fill every queue
                    pt[0] = kb;
                    q_step<NS, QP, G, T, 0>(m, q, true);
                    QMem<NS, T, FORM, S> qm{m, q};
                    NS::template body_slice<FORM, S>(qm, args.s, pt);
                }
                // steady state: straight-line shift + one load per queue, so the
                // unrolled planes' loads can all be issued ahead
#pragma unroll UNR
                for (int k = kb + 1; k < ke; ++k) {
                    pt[0] = k;
                    q_step<NS, QP, G, T, 0>(m, q, false);
                    QMem<NS, T, FORM, S> qm{m, q};
                    NS::template body_slice<FORM, S>(qm, args.s, pt);
                }
            } else {
#pragma unroll UNR
                for (int k = kb; k < ke; ++k) {
                    pt[0] = k;
                    NS::template body_slice<FORM, S>(m, args.s, pt);
                }
            }
        } else {
            march_slice<NS, T, FORM, S + 1, UNR>(m, args, pt, slice, kb, ke);
        }
    }
}

template <class NS, class T, int FORM, int BX, int BY, int UNR>
__global__ void __launch_bounds__(BX* BY) sliced_kernel(const __grid_constant__ KernelArgs<NS> args, int kchunk) {
    static_assert(NS::NLOOP == 3, "sliced skeleton: 3-D nests");
    constexpr int NSL = NS::nslices[FORM];
    const int slice = (int)(blockIdx.z % NSL);
    const int chunk = (int)(blockIdx.z / NSL);
    // x tiles start at a 128-byte-aligned column (x0 = lo aligned down), so a
    // 32-byte sector of a stored row is written by one CTA only
    const int xlo = (int)args.lo[2];
    const int x0 = xlo - (((xlo % 16) + 16) % 16);
    const int x = x0 + (int)(blockIdx.x * BX + threadIdx.x);
    const int y = args.lo[1] + (int)(blockIdx.y * BY + threadIdx.y);
    if (x < xlo || x >= args.hi[2] || y >= args.hi[1]) return;
    const int kb = args.lo[0] + chunk * kchunk;
    const int ke = min(kb + kchunk, (int)args.hi[0]);
    int pt[3];
    pt[1] = y;
    pt[2] = x;
    NaiveMem<NS, T, FORM == ACS_ORIGINAL> m{args, pt};
    march_slice<NS, T, FORM, 0, UNR>(m, args, pt, slice, kb, ke);
    if (args.sh.enabled) __threadfence_system();   // peer write-through visible before the step flag
}

template <class NS, class T, int FORM, int BX, int BY, int KCH, int UNR>
acs_status launch_sliced(const LaunchReq& r) {
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    constexpr int NSL = NS::nslices[FORM];
    const long long x0 = ka.lo[2] - (((ka.lo[2] % 16) + 16) % 16);
    const long long nx = ka.hi[2] - x0, ny = ka.hi[1] - ka.lo[1], nz = ka.hi[0] - ka.lo[0];
    const long long chunks = (nz + KCH - 1) / KCH;
    dim3 grid((unsigned)((nx + BX - 1) / BX), (unsigned)((ny + BY - 1) / BY), (unsigned)(chunks * NSL));
    if (r.preload) return preload_fn((const void*)sliced_kernel<NS, T, FORM, BX, BY, UNR>);
    sliced_kernel<NS, T, FORM, BX, BY, UNR><<<grid, dim3(BX, BY, 1), 0, r.stream>>>(ka, KCH);
    return check_launch("sliced");
}

template <class NS, class T, int BX, int BY, int KCH, int UNR = 4>
void fill_sliced(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_sliced<NS, T, 0, BX, BY, KCH, UNR>;
    e.launch[prec][1][slot] = &launch_sliced<NS, T, 1, BX, BY, KCH, UNR>;
    e.launch[prec][2][slot] = &launch_sliced<NS, T, 2, BX, BY, KCH, UNR>;
    e.launch[prec][3][slot] = &launch_sliced<NS, T, 3, BX, BY, KCH, UNR>;
    e.launch[prec][4][slot] = &launch_sliced<NS, T, 4, BX, BY, KCH, UNR>;
    e.sched_name[prec][slot] = "sliced " + std::to_string(NS::nslices[4]) + " components, block " +
                               std::to_string(BX) + "x" + std::to_string(BY) + ", k-chunk " + std::to_string(KCH) +
                               ", unroll " + std::to_string(UNR);
    for (int v = 0; v < 5; ++v)
        if (e.best[prec][v] == 0 && v != ACS_ORIGINAL) e.best[prec][v] = slot;
}

}  // namespace acs
