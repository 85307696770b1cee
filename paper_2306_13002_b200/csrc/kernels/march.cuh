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
template <class NS, class T, int LAYOUT, int TX, int TY, int RX = 1>
struct MarchPlan {
    static constexpr int NL = NS::NLOOP;
    static constexpr int X = NL - 1;   // loop index of the innermost loop (tile x)
    static constexpr int Y = NL == 3 ? 1 : -9;
    // RX > 1 (register windows): the tile origin is aligned down to a 16-byte
    // element multiple V and every staged array's box starts RA elements
    // below it (RA = the largest x reach below the point, rounded up to V), so
    // a thread's point group and every window row sit at compile-time-known
    // alignment.
    static constexpr bool ALIGNED = RX > 1;
    static constexpr int V = 16 / (int)sizeof(T);
    static constexpr int ra() {
        int r = 0;
        for (int a = 0; a < NS::NARR; ++a)
            if (NS::stageable(a))
                for (int p = 0; p < NS::ndim(a); ++p)
                    if (NS::ld_sig(a, p) == X && -NS::ld_lo(a, p) > r) r = -NS::ld_lo(a, p);
        return (r + V - 1) / V * V;
    }
    static constexpr int RA = ra();
    // box origin of array a at position p, relative to the tile's point
    static constexpr int lo(int a, int p) { return ALIGNED && NS::ld_sig(a, p) == X ? -RA : NS::ld_lo(a, p); }

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
        const int w = NS::ld_hi(a, p) - lo(a, p);
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
        const int need = inner_is_x(a) && !ALIGNED ? e + q - 1 : e;
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
    // x-origin shift of the tensor maps (elements, the same for every staged
    // array): an array whose data pointer is not 16-byte aligned (a
    // sector-aligned native row offset) is described from the aligned address
    // adjx elements earlier, so its tensor x coordinate is x + adjx
    int adjx;
    // ring arrays read exactly once (no halo, span 1) loaded with an L2 evict_first
    // policy (bit a); ACS_TMA_EVICT=1 turns it on (an experiment knob, tools/gpu)
    unsigned evict;
};

// per-CTA state a body's memory policy needs
template <class NS, class T, int LAYOUT, int TX, int TY, int PF, int RX = 1>
struct MarchMem {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY, RX>;
    static constexpr int D = P::maxspan() + PF;
    using value_t = T;
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
                const int l = off[p] - P::lo(ARR, p);
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

    // start of unique window K (WinPlan) in its staged box; lx0 / ly0 = the
    // thread's first point (aligned-origin path: alignment shift 0)
    template <class WP, int K>
    __device__ __forceinline__ const T* uwin_ptr(int lx0, int ly0) const {
        constexpr int A = WP::PL.u[K].arr;
        int idx = 0;
        int delta = D;
#pragma unroll
        for (int p = 0; p < NS::ndim(A); ++p) {
            const int s = NS::ld_sig(A, p);
            const int o = s == P::X ? WP::PL.u[K].xlo : WP::u_off(K, p);
            const int l = o - P::lo(A, p);
            if (s == 0) delta = D + o - NS::ld_hi(A, p);
            else if (s == P::X) idx += (lx0 + l) * P::bstride(A, p);
            else if (s == P::Y) idx += (ly0 + l) * P::bstride(A, p);
            else idx += l * P::bstride(A, p);
        }
        if (delta >= D) delta -= D;
        return reinterpret_cast<const T*>(box_base<A>(delta)) + idx;
    }

    // a data-dependent index whose every candidate value is affine in the loop
    // variables (the lowering's value-set proof): the staged box was sized to
    // hold all of them, so no range check and no global fallback
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx_in(I... ii) const {
        if constexpr (P::staged(ARR)) {
            const int v[sizeof...(I)] = {(int)ii...};
            int idx = 0, delta = 0;
#pragma unroll
            for (int p = 0; p < (int)sizeof...(I); ++p) {
                const int s = NS::ld_sig(ARR, p);
                const int lo = P::lo(ARR, p);
                if (s == 0) {
                    delta = D + (v[p] - k) - NS::ld_hi(ARR, p);
                } else {
                    const int l = v[p] - lo - (s == P::X ? orgx : (s == P::Y ? orgy : 0));
                    idx += (l + (s == P::X ? sh[ARR] : 0)) * P::bstride(ARR, p);
                }
            }
            if (delta >= D) delta -= D;
            return box_base<ARR>(delta)[idx];
        } else {
            return g.template ldx<ARR>(ii...);
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
                const int lo = P::lo(ARR, p);
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

// ---- register windows: 2.5-D register blocking ------------------------------
//
// A thread owns NY = TY/BY adjacent rows x RX adjacent x points of the tile.
// Per march step it needs, for every static-load ROW of the body (the
// lowering's row table: array + subscript offsets, innermost x aside) and
// every one of its rows, a window of consecutive x elements.  The planner
// (constexpr, per form) merges them into UNIQUE windows keyed by (array,
// absolute y, march offset dz, other offsets) — the j+1 row of thread row 0
// is the centre row of thread row 1 — and marks a window QUEUED when the
// window one plane further along the march (dz + 1) covers its x range:
// the value it needs at step s+1 is already in registers at step s.  Only
// the rest is read from the staged TMA boxes, as 16-byte LDS.128 at
// compile-time alignment (the tile origin is aligned down to V = 16/sizeof(T)
// elements and every box starts RA below it).  jacobi7 (2 rows x 2 points per
// thread): 3.5 doubles of shared memory per point instead of 7; wave4: the
// k-2 / k-1 / k+1 planes of u come from the queue.
//
// Stores of arrays the nest never loads are deferred per point group and
// written as one 16-byte STG per V points.
struct UWin {
    int arr = -1;
    int off[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // x position 0, y position = absolute thread row offset
    int xlo = 0, xhi = 0;
    int src = -1;                             // queued: copied from this window at the end of a step
    int dz = 0;
};

template <int MAXU, int MAXR, int NYM>
struct UPlan {
    UWin u[MAXU];
    int n = 0;
    int rmap[MAXR][NYM] = {};
    int woff[MAXU + 1] = {};
    int order[MAXU] = {};
    bool ok = true;
};

template <class NS, class T, int LAYOUT, int TX, int TY, int BY, int FORM, int RX>
struct WinPlan {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY, RX>;
    static constexpr int V = 16 / (int)sizeof(T);
    static constexpr int NY = TY / BY;
    static constexpr int RXV = RX / V;
    static constexpr int MAXR = NS::NROW > 0 ? NS::NROW : 1;
    static constexpr int MAXU = MAXR * NY;
    static constexpr int pos_of(int a, int sg) {
        for (int p = 0; p < NS::ndim(a); ++p)
            if (NS::ld_sig(a, p) == sg) return p;
        return -1;
    }
    static constexpr int xpos(int a) { return pos_of(a, P::X); }
    static constexpr bool row_on(int r) {
        return ((NS::row_forms(r) >> FORM) & 1) && P::staged(NS::row_arr(r)) && xpos(NS::row_arr(r)) >= 0 &&
               !NS::is_int(NS::row_arr(r));
    }
    static constexpr UPlan<MAXU, MAXR, NY> build() {
        UPlan<MAXU, MAXR, NY> pl{};
        for (int r = 0; r < NS::NROW; ++r) {
            if (!row_on(r)) continue;
            const int a = NS::row_arr(r), xp = xpos(a), yp = pos_of(a, P::Y), mp = pos_of(a, 0);
            for (int ry = 0; ry < NY; ++ry) {
                int off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int p = 0; p < NS::ndim(a); ++p)
                    off[p] = p == xp ? 0 : (p == yp ? NS::row_off(r, p) + ry : NS::row_off(r, p));
                int k = -1;
                for (int j = 0; j < pl.n && k < 0; ++j) {
                    bool same = pl.u[j].arr == a;
                    for (int p = 0; p < 8; ++p) same = same && pl.u[j].off[p] == off[p];
                    if (same) k = j;
                }
                if (k < 0) {
                    if (pl.n >= MAXU) {
                        pl.ok = false;
                        return pl;
                    }
                    k = pl.n++;
                    pl.u[k].arr = a;
                    for (int p = 0; p < 8; ++p) pl.u[k].off[p] = off[p];
                    pl.u[k].xlo = NS::row_xlo(r);
                    pl.u[k].xhi = NS::row_xhi(r);
                    pl.u[k].dz = mp >= 0 ? off[mp] : 0;
                } else {
                    if (NS::row_xlo(r) < pl.u[k].xlo) pl.u[k].xlo = NS::row_xlo(r);
                    if (NS::row_xhi(r) > pl.u[k].xhi) pl.u[k].xhi = NS::row_xhi(r);
                }
                pl.rmap[r][ry] = k;
            }
        }
        for (int k = 0; k < pl.n; ++k) {
            const int a = pl.u[k].arr, mp = pos_of(a, 0);
            if (mp < 0) continue;
            for (int j = 0; j < pl.n; ++j) {
                if (pl.u[j].arr != a || pl.u[j].off[mp] != pl.u[k].off[mp] + 1) continue;
                bool same = true;
                for (int p = 0; p < 8; ++p) same = same && (p == mp || pl.u[j].off[p] == pl.u[k].off[p]);
                if (same && pl.u[j].xlo <= pl.u[k].xlo && pl.u[j].xhi >= pl.u[k].xhi) pl.u[k].src = j;
            }
        }
        for (int k = 0; k < pl.n; ++k) pl.woff[k + 1] = pl.woff[k] + RX + pl.u[k].xhi - pl.u[k].xlo;
        // queue copies in increasing dz: a source is read before it is overwritten
        int m = 0;
        for (int dz = -64; dz <= 64; ++dz)
            for (int k = 0; k < pl.n; ++k)
                if (pl.u[k].dz == dz) pl.order[m++] = k;
        return pl;
    }
    static constexpr UPlan<MAXU, MAXR, NY> PL = build();
    // runtime-index accessors usable in device code (a local constant copy)
    static __host__ __device__ constexpr int u_off(int k, int p) {
        constexpr UPlan<MAXU, MAXR, NY> pl = build();
        return pl.u[k].off[p];
    }
    static constexpr int total() { return PL.woff[PL.n]; }
    static constexpr int width(int k) { return RX + PL.u[k].xhi - PL.u[k].xlo; }
    static constexpr int align(int k) {   // misalignment (elements) of window k's start in its box row
        const int m = PL.u[k].xlo - P::lo(PL.u[k].arr, xpos(PL.u[k].arr));
        return ((m % V) + V) % V;
    }
    template <int ARR, int... O>
    static constexpr int row_of() {
        constexpr int off[sizeof...(O)] = {O...};
        for (int r = 0; r < NS::NROW; ++r) {
            if (NS::row_arr(r) != ARR || !row_on(r)) continue;
            bool ok = true;
            for (int p = 0; p < (int)sizeof...(O); ++p)
                if (p != xpos(ARR) && NS::row_off(r, p) != off[p]) ok = false;
            if (ok) return r;
        }
        return -1;
    }
    // deferred vector stores: static store targets of arrays the nest never
    // loads, at an x offset that keeps the point group 16-byte aligned
    static constexpr int sxpos(int a) {
        for (int p = 0; p < NS::ndim(a); ++p)
            if (NS::sig(a, p) == P::X) return p;
        return -1;
    }
    static constexpr bool srow_on(int r) {
        const int a = NS::srow_arr(r);
        return ((NS::srow_forms(r) >> FORM) & 1) && !NS::is_loaded(a) && !NS::is_int(a) && sxpos(a) >= 0 &&
               NS::srow_off(r, sxpos(a)) % V == 0;
    }
    static constexpr int soff(int r) {
        int o = 0;
        for (int b = 0; b < r; ++b)
            if (srow_on(b)) o += RX;
        return o;
    }
    static constexpr int stotal() { return soff(NS::NSROW); }
    template <int ARR, int... O>
    static constexpr int srow_of() {
        constexpr int off[sizeof...(O)] = {O...};
        for (int r = 0; r < NS::NSROW; ++r) {
            if (NS::srow_arr(r) != ARR || !srow_on(r)) continue;
            bool ok = true;
            for (int p = 0; p < (int)sizeof...(O); ++p)
                if (NS::srow_off(r, p) != off[p]) ok = false;
            if (ok) return r;
        }
        return -1;
    }
    template <int R, class G, int... PP>
    static __device__ __forceinline__ long long sidx(const G& g, std::integer_sequence<int, PP...>) {
        return g.template static_index<NS::srow_arr(R), NS::srow_off(R, PP)...>();
    }
    static constexpr bool usable() {
        if (RX <= 1) return false;
        if (LAYOUT != 0 || RX % V != 0 || TX % RX != 0 || NS::NROW > 64) return false;
        return PL.ok && total() > 0 && total() + NY * stotal() <= 192;
    }
};

// per-point view of the windows: point (RY, R0) of the thread's group
template <class MM, class WP, class NS, int RY, int R0>
struct WinMem {
    const MM& m;
    const typename MM::value_t* win;
    typename MM::value_t* out;     // deferred stores of this thread row
    bool defer;
    template <int ARR>
    using elem_t = typename MM::template elem_t<ARR>;
    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const {
        constexpr int r = WP::template row_of<ARR, O...>();
        if constexpr (r >= 0) {
            constexpr int off[sizeof...(O)] = {O...};
            constexpr int ox = off[WP::xpos(ARR)];
            constexpr int k = WP::PL.rmap[r][RY];
            constexpr int idx = WP::PL.woff[k] + R0 + ox - WP::PL.u[k].xlo;
            return win[idx];
        } else {
            return m.template ld<ARR, O...>();
        }
    }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... ii) const { return m.template ldx<ARR>(ii...); }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx_in(I... ii) const { return m.template ldx_in<ARR>(ii...); }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const {
        constexpr int r = WP::template srow_of<ARR, O...>();
        if constexpr (r >= 0) {
            if (defer) {
                out[WP::soff(r) + R0] = v;
                return;
            }
        }
        m.template st<ARR, O...>(v);
    }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const { m.template stx<ARR>(args...); }
};

template <class T>
struct Vec16;
template <>
struct Vec16<float> {
    using type = float4;
};
template <>
struct Vec16<double> {
    using type = double2;
};

template <class P, class NS>
__host__ __device__ constexpr int xshift(int a, int orgx) {
    if (P::ALIGNED || !P::inner_is_x(a)) return 0;
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
                    else if (s == P::X)
                        c[d] = orgx + P::lo(A, p) - (d == 0 ? xshift<P, NS>(A, orgx) : 0);
                    else if (s == P::Y) c[d] = orgy + NS::ld_lo(A, p);
                    else c[d] = NS::ld_lo(A, p);
                }
                unsigned char* dst = P::on_ring(A) ? slot_base + P::ring_off(A) : stat + P::static_off(A);
                if ((maps.evict >> A) & 1u)
                    tma_load_hint<NS::ndim(A)>(dst, &maps.m[A], c, bar, l2_evict_first_policy());
                else
                    tma_load<NS::ndim(A)>(dst, &maps.m[A], c, bar);
            }
        }
        march_issue<P, NS, A + 1>(slot_base, maps, bar, plane_base, orgx, orgy, want_static, stat);
    }
}

// ---- one point per thread column (RX == 1): hoisted addressing ---------------
//
// Everything about a thread's points that does not change along the march is
// computed once per thread: its element offset inside every staged box and
// its global address in every statically stored (or unstaged loaded) array.
// Per march step only the shared-memory address of each ring plane the body
// reads (one add per array and plane) and the global pointers (one add per
// array) move; the body's static loads are then one LDS at a compile-time byte
// offset and its stores one STG at a per-thread constant offset — instead of
// re-deriving the ring slot, the box index and a 64-bit subscript product per
// load and store of every point (jacobi7: 74 -> see profiles/r02_jacobi.md).
template <class NS, class T, class P, int MS>
struct FastState {
    unsigned plane[NS::NARR][MS > 0 ? MS : 1];   // byte offset (from the ring) of the thread's first point, per plane
    unsigned stat[NS::NARR];                     // same in the static (plane-less) boxes
    char* gp[NS::NARR];                          // global address of the thread's first point at plane k
    long long gstep[NS::NARR];                   // bytes per march step

    // arrays the body stores with static subscripts in form FORM
    static constexpr bool stored_static(int a, int form) {
        for (int r = 0; r < NS::NSROW; ++r)
            if (NS::srow_arr(r) == a && ((NS::srow_forms(r) >> form) & 1)) return true;
        return false;
    }
    static constexpr bool needs_gp(int a, int form) {
        return stored_static(a, form) || (!P::staged(a) && NS::is_loaded(a));
    }
    // the body of form `form` reads array a at the thread's own inner
    // coordinates in march plane dz (a static-load row with every non-march
    // offset 0 whose x range covers 0)
    static constexpr bool column(int a, int dz, int form) {
        const int mp = P::march_pos(a);
        for (int r = 0; r < NS::NROW; ++r) {
            if (NS::row_arr(r) != a || !((NS::row_forms(r) >> form) & 1)) continue;
            if (NS::row_xlo(r) > 0 || NS::row_xhi(r) < 0) continue;
            bool ok = NS::row_off(r, mp) == dz;
            for (int p = 0; p < NS::ndim(a); ++p)
                if (p != mp && NS::row_off(r, p) != 0) ok = false;
            if (ok) return true;
        }
        return false;
    }
    // every load of the body comes from a staged box (no global, no dynamic
    // index): a point outside the domain can run the body on in-box values
    // and just skip its stores — no branch per point
    static constexpr bool all_staged() {
        if (NS::has_dynamic_index) return false;
        for (int a = 0; a < NS::NARR; ++a)
            if (NS::is_loaded(a) && !P::staged(a)) return false;
        return true;
    }
    // k-column register queue: a ring array whose column the body reads in its
    // top plane and in at least one lower plane — the lower planes' values were
    // read as the top plane of earlier steps and stay in registers
    // lowest march plane of array a the body reads from SHARED memory in form
    // `form`: every plane for unqueued arrays; for queued ones the planes of
    // their non-column loads (rows off the thread's own column) and the top
    // plane that feeds the queue — lower column planes live in registers
    static constexpr int smem_lo(int a, int form) {
        const int mp = P::march_pos(a);
        if (!queued(a, form)) return NS::ld_lo(a, mp);
        int lo = NS::ld_hi(a, mp);
        for (int r = 0; r < NS::NROW; ++r) {
            if (NS::row_arr(r) != a || !((NS::row_forms(r) >> form) & 1)) continue;
            bool col = NS::row_xlo(r) == 0 && NS::row_xhi(r) == 0;
            for (int p = 0; p < NS::ndim(a); ++p)
                if (p != mp && NS::row_off(r, p) != 0) col = false;
            if (!col && NS::row_off(r, mp) < lo) lo = NS::row_off(r, mp);
        }
        return lo;
    }
    // ring planes the hoisted path needs resident: the deepest shared-memory
    // reach of any staged array (the queue prologue still reads the full span
    // once, at step 0, so the ring never holds fewer bundles than the span)
    static constexpr int smem_span(int form) {
        int m = 1;
        for (int a = 0; a < NS::NARR; ++a)
            if (P::on_ring(a)) {
                const int sp = NS::ld_hi(a, P::march_pos(a)) - smem_lo(a, form) + 1;
                if (sp > m) m = sp;
            }
        return m;
    }
    static constexpr bool queued(int a, int form) {
        if (!P::on_ring(a) || P::span(a) < 2 || NS::is_int(a)) return false;
        const int mp = P::march_pos(a);
        if (!column(a, NS::ld_hi(a, mp), form)) return false;
        for (int dz = NS::ld_lo(a, mp); dz < NS::ld_hi(a, mp); ++dz)
            if (column(a, dz, form)) return true;
        return false;
    }
};

template <class MM, class FS, class NS, class P, int FORM, int PX, int PY, int PI, int NPTS>
struct FastPt {
    const MM& m;
    const FS& fs;
    typename MM::value_t (*q)[NPTS][P::maxspan() > 0 ? P::maxspan() : 1];   // [array][point][plane] queue
    bool act;                                                                // the point is in the domain
    template <int ARR>
    using elem_t = typename MM::template elem_t<ARR>;

    template <int ARR, int... O>
    static constexpr int box_const() {   // element offset of this load relative to the thread's first point
        constexpr int off[sizeof...(O)] = {O...};
        int c = 0;
        for (int p = 0; p < (int)sizeof...(O); ++p) {
            const int s = NS::ld_sig(ARR, p);
            if (s == 0) continue;
            if (s == P::X) c += (off[p] + PX) * P::bstride(ARR, p);
            else if (s == P::Y) c += (off[p] + PY) * P::bstride(ARR, p);
            else c += (off[p] - P::lo(ARR, p)) * P::bstride(ARR, p);
        }
        return c;
    }
    template <int ARR, int... O>
    static constexpr int plane_of() {
        constexpr int off[sizeof...(O)] = {O...};
        for (int p = 0; p < (int)sizeof...(O); ++p)
            if (NS::ld_sig(ARR, p) == 0) return off[p] - NS::ld_lo(ARR, p);
        return 0;
    }
    template <int ARR, int... O>
    __device__ __forceinline__ long long gconst() const {   // global element offset (runtime strides)
        constexpr int off[sizeof...(O)] = {O...};
        long long c = 0;
#pragma unroll
        for (int p = 0; p < (int)sizeof...(O); ++p) {
            const int s = NS::sig(ARR, p);
            const int o = off[p] + (s == P::X ? PX : (s == P::Y ? PY : 0));
            if (o != 0) c += (long long)o * m.g.a.arr[ARR].stride[p];
        }
        return c;
    }

    template <int ARR, int... O>
    static constexpr bool at_column() {
        constexpr int off[sizeof...(O)] = {O...};
        for (int p = 0; p < (int)sizeof...(O); ++p)
            if (NS::ld_sig(ARR, p) != 0 && off[p] != 0) return false;
        return true;
    }

    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const {
        if constexpr (FS::queued(ARR, FORM) && at_column<ARR, O...>()) {
            constexpr int i = plane_of<ARR, O...>();
            if constexpr (i < P::span(ARR) - 1) {
                return q[ARR][PI][i];                    // read as the top plane of an earlier step
            } else {
                const elem_t<ARR> v = *reinterpret_cast<const elem_t<ARR>*>(
                    m.ring + fs.plane[ARR][i] + box_const<ARR, O...>() * (int)sizeof(elem_t<ARR>));
                q[ARR][PI][i] = v;
                return v;
            }
        } else if constexpr (P::staged(ARR)) {
            constexpr int c = box_const<ARR, O...>() * (int)sizeof(elem_t<ARR>);
            const unsigned b = P::on_ring(ARR) ? fs.plane[ARR][plane_of<ARR, O...>()] : fs.stat[ARR];
            return *reinterpret_cast<const elem_t<ARR>*>(m.ring + b + c);
        } else if constexpr (FS::needs_gp(ARR, FORM)) {
            const elem_t<ARR>* p = reinterpret_cast<const elem_t<ARR>*>(fs.gp[ARR]) + gconst<ARR, O...>();
            if constexpr (NS::readonly(ARR)) return ld_ro(p);
            else return ld_plain(p);
        } else {
            return m.template ld<ARR, O...>();
        }
    }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... ii) const { return m.template ldx<ARR>(ii...); }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx_in(I... ii) const { return m.template ldx_in<ARR>(ii...); }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const {
        if (!act) return;
        if constexpr (FS::stored_static(ARR, FORM)) {
            // sharded launch: only planes within reach of a slab face take the
            // write-through path (a CTA-uniform test per step)
            bool fast = !m.g.a.sh.enabled;
            if (!fast) {
                constexpr int off[sizeof...(O)] = {O...};
                constexpr int o0 = NS::sig(ARR, 0) == 0 ? off[0] : 0;
                const long long g = (long long)m.k + o0 + m.g.a.sh.origin;
                fast = NS::sig(ARR, 0) == 0 && g >= m.g.a.sh.lo_thr && g < m.g.a.sh.hi_thr;
            }
            if (fast) {
                *(reinterpret_cast<elem_t<ARR>*>(fs.gp[ARR]) + gconst<ARR, O...>()) = v;
                return;
            }
        }
        m.template st<ARR, O...>(v);   // write-through path
    }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const { m.template stx<ARR>(args...); }
};

// a thread's points: NPX along x strided by the block width (coalesced rows),
// NPY ADJACENT rows (their shared y-neighbour rows are one LDS each)
template <class NS, class P, class MM, class FS, int FORM, int NPX, int NPY, int BX, int I, class Q>
__device__ __forceinline__ void fast_points(MM& m, const FS& fs, Q q, const KernelArgs<NS>& args, int* pt,
                                            const bool* inb, int x0, int y0, int lx0, int ly0) {
    if constexpr (I < NPX * NPY) {
        constexpr int rx = I % NPX, ry = I / NPX;
        if (FS::all_staged() || inb[I]) {
            pt[P::X] = x0 + rx * BX;
            if constexpr (NS::NLOOP == 3) pt[1] = y0 + ry;
            if constexpr (NS::has_dynamic_index) {
                m.lx = lx0 + rx * BX;
                m.ly = ly0 + ry;
            }
            FastPt<MM, FS, NS, P, FORM, rx * BX, ry, I, NPX * NPY> fp{m, fs, q, inb[I]};
            NS::template body<FORM>(fp, args.s, pt);
        }
        fast_points<NS, P, MM, FS, FORM, NPX, NPY, BX, I + 1>(m, fs, q, args, pt, inb, x0, y0, lx0, ly0);
    }
}

// prologue of the k-column queue: the lower planes of step 0 from the ring
template <class NS, class P, class FS, int FORM, int NPX, int NPY, int BX, int A, class T, class Q>
__device__ __forceinline__ void fast_queue_fill(const unsigned char* ring, const FS& fs, Q q, int b) {
    if constexpr (A < NS::NARR) {
        if constexpr (FS::queued(A, FORM)) {
            constexpr int mp = P::march_pos(A);
            int xo = 0;   // box element offset of the column (0, 0) relative to the thread's first point
#pragma unroll
            for (int p = 0; p < NS::ndim(A); ++p)
                if (p != mp && NS::ld_sig(A, p) != P::X && NS::ld_sig(A, p) != P::Y)
                    xo += (0 - P::lo(A, p)) * P::bstride(A, p);
#pragma unroll
            for (int I = 0; I < NPX * NPY; ++I) {
                const int rx = I % NPX, ry = I / NPX;
                int c = xo;
#pragma unroll
                for (int p = 0; p < NS::ndim(A); ++p) {
                    if (NS::ld_sig(A, p) == P::X) c += rx * BX * P::bstride(A, p);
                    else if (NS::ld_sig(A, p) == P::Y) c += ry * P::bstride(A, p);
                }
#pragma unroll
                for (int i = 0; i < P::span(A) - 1; ++i)
                    if (P::maxspan() - P::span(A) + i == b)   // plane i of array A arrives in bundle b
                        q[A][I][i] = *reinterpret_cast<const T*>(ring + fs.plane[A][i] + c * (int)sizeof(T));
            }
        }
        fast_queue_fill<NS, P, FS, FORM, NPX, NPY, BX, A + 1, T>(ring, fs, q, b);
    }
}

// end of step: the queue moves one plane along the march
template <class NS, class P, class FS, int FORM, int NPTS, int A, class Q>
__device__ __forceinline__ void fast_queue_shift(Q q) {
    if constexpr (A < NS::NARR) {
        if constexpr (FS::queued(A, FORM)) {
#pragma unroll
            for (int I = 0; I < NPTS; ++I)
#pragma unroll
                for (int i = 0; i + 1 < P::span(A); ++i) q[A][I][i] = q[A][I][i + 1];
        }
        fast_queue_shift<NS, P, FS, FORM, NPTS, A + 1>(q);
    }
}

// TX x TY points per tile, BX x BY threads: each thread computes (TX/BX) x (TY/BY)
// points per march step, amortising the step's barrier / mbarrier wait.
template <class WP, class MM, class NS, int FORM, int RY, int R0, int RX>
__device__ __forceinline__ void win_run(MM& m, const typename MM::value_t* win, typename MM::value_t* out,
                                        bool defer, const KernelArgs<NS>& args, int* pt, int lx0, int xlo, int xhi) {
    if constexpr (R0 < RX) {
        const int x = m.orgx + lx0 + R0;
        if (x < xhi && x >= xlo) {
            pt[NS::NLOOP - 1] = x;
            m.lx = lx0 + R0;
            WinMem<MM, WP, NS, RY, R0> wm{m, win, out, defer};
            NS::template body<FORM>(wm, args.s, pt);
        }
        win_run<WP, MM, NS, FORM, RY, R0 + 1, RX>(m, win, out, defer, args, pt, lx0, xlo, xhi);
    }
}

// one thread row's deferred stores: one 16-byte vector store per V points
template <class WP, class MM, class NS, int R>
__device__ __forceinline__ void win_flush(const MM& m, const typename MM::value_t* out) {
    if constexpr (R < NS::NSROW) {
        if constexpr (WP::srow_on(R)) {
            using E = typename MM::value_t;
            using VT = typename Vec16<E>::type;
            constexpr int A = NS::srow_arr(R);
            const long long idx = WP::template sidx<R>(m.g, std::make_integer_sequence<int, NS::ndim(A)>{});
            E* p = reinterpret_cast<E*>(m.g.a.arr[A].base) + idx;
#pragma unroll
            for (int v = 0; v < WP::RXV; ++v)
                *reinterpret_cast<VT*>(p + v * WP::V) = *reinterpret_cast<const VT*>(&out[WP::soff(R) + v * WP::V]);
        }
        win_flush<WP, MM, NS, R + 1>(m, out);
    }
}

// unique window K from its staged box (skipped for queued windows after the
// first step of a chunk: they were copied at the end of the previous step)
template <class WP, class MM, class NS, int K>
__device__ __forceinline__ void win_load(const MM& m, typename MM::value_t* win, int lx0, int ly0, bool first) {
    if constexpr (K < WP::PL.n) {
        constexpr bool queued = WP::PL.u[K].src >= 0;
        constexpr int base = WP::PL.woff[K];
        if (first || !queued) {
            using E = typename MM::value_t;
            using VT = typename Vec16<E>::type;
            constexpr int V = WP::V, A = WP::align(K), W = WP::width(K);
            constexpr int NV = (A + W + V - 1) / V;
            const E* p = m.template uwin_ptr<WP, K>(lx0, ly0) - A;
            E tmp[NV * V];
#pragma unroll
            for (int v = 0; v < NV; ++v) *reinterpret_cast<VT*>(&tmp[v * V]) = *reinterpret_cast<const VT*>(p + v * V);
#pragma unroll
            for (int w = 0; w < W; ++w) win[base + w] = tmp[A + w];
        }
        win_load<WP, MM, NS, K + 1>(m, win, lx0, ly0, first);
    }
}

// end of step: shift the queued windows one plane along the march
template <class WP, class E, int I>
__device__ __forceinline__ void win_shift(E* win) {
    if constexpr (I < WP::PL.n) {
        constexpr int K = WP::PL.order[I];
        constexpr int S = WP::PL.u[K].src;
        if constexpr (S >= 0) {
            constexpr int dst = WP::PL.woff[K];
            constexpr int src = WP::PL.woff[S] + WP::PL.u[K].xlo - WP::PL.u[S].xlo;
            constexpr int W = WP::width(K);
#pragma unroll
            for (int w = 0; w < W; ++w) win[dst + w] = win[src + w];
        }
        win_shift<WP, E, I + 1>(win);
    }
}

template <class WP, class M, class NS, int FORM, int RY, int RX, class T>
__device__ __forceinline__ void win_rows(M& m, const T* win, bool vec_ok, const KernelArgs<NS>& args, int* pt,
                                         int lx0, int ly0, int xlo0, int orgy) {
    if constexpr (RY < WP::NY) {
        using P = typename WP::P;
        const int y = orgy + ly0 + RY;
        if (NS::NLOOP < 3 || y < args.hi[1]) {
            m.ly = ly0 + RY;
            if constexpr (NS::NLOOP == 3) pt[1] = y;
            T out[WP::stotal() > 0 ? WP::stotal() : 1];
            const int x0 = m.orgx + lx0;
            bool defer = vec_ok && x0 >= xlo0 && x0 + RX <= args.hi[P::X];
            if (args.sh.enabled) {
                // write-through to a neighbour happens in the scalar store path:
                // keep it for planes within reach of the slab faces
                const long long g = (long long)pt[0] + args.sh.origin;
                if (g < args.sh.lo_thr + 4 || g >= args.sh.hi_thr - 4) defer = false;
            }
            win_run<WP, M, NS, FORM, RY, 0, RX>(m, win, out, defer, args, pt, lx0, xlo0, args.hi[P::X]);
            if constexpr (WP::stotal() > 0) {
                if (defer) {
                    pt[P::X] = x0;
                    win_flush<WP, M, NS, 0>(m, out);
                }
            }
        }
        win_rows<WP, M, NS, FORM, RY + 1, RX>(m, win, vec_ok, args, pt, lx0, ly0, xlo0, orgy);
    }
}

// ring depth of a march kernel: span + PF bundles; on the hoisted 3-D path the
// k-column queue keeps the lower column planes in registers, so only the
// planes read from shared memory count (the queue prologue consumes the lower
// bundles one by one and recycles their slots).  wave4 u: 5 + PF -> 3 + PF.
template <class NS, class T, int LAYOUT, int TX, int TY, int RX, int PF, int FORM>
constexpr int march_ring_depth() {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY, RX>;
    constexpr int MS = P::maxspan();
    if constexpr (RX == 1 && NS::NLOOP == 3) {
        return FastState<NS, T, P, MS>::smem_span(FORM) + PF;
    } else {
        return MS + PF;
    }
}

template <class NS, class T, int FORM, int LAYOUT, int TX, int TY, int BX, int BY, int PF, int RX = 1>
__global__ void __launch_bounds__(BX* BY) march_kernel(const __grid_constant__ KernelArgs<NS> args,
                                                       const __grid_constant__ TmaMaps<NS> maps, int kchunk) {
    static_assert(TX % BX == 0 && TY % BY == 0, "tile must be a multiple of the block");
    static_assert(RX == 1 || TX == BX * RX, "register windows: one RX group of adjacent points per thread");
    using P = MarchPlan<NS, T, LAYOUT, TX, TY, RX>;
    using M = MarchMem<NS, T, LAYOUT, TX, TY, PF, RX>;
    constexpr int D = march_ring_depth<NS, T, LAYOUT, TX, TY, RX, PF, FORM>();
    static_assert(RX == 1 && NS::NLOOP == 3 || D == M::D, "generic path: the ring depth MarchMem assumes");
    constexpr int MS = P::maxspan();
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem;
    unsigned char* stat = smem + D * P::slot_bytes();
    uint64_t* bars = reinterpret_cast<uint64_t*>(stat + P::static_bytes());   // D ring + 1 static

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * BX + tx;
    const int xlo0 = (int)args.lo[P::X];
    // aligned origin: orgx + adj (the tensor-map x coordinate) is a multiple of V
    const int orgx = (P::ALIGNED ? xlo0 - ((((xlo0 + maps.adjx) % P::V) + P::V) % P::V) : xlo0) + blockIdx.x * TX;
    const int orgy = NS::NLOOP == 3 ? args.lo[1] + blockIdx.y * TY : 0;
    const int kb = args.lo[0] + blockIdx.z * kchunk;
    const int ke = min(kb + kchunk, args.hi[0]);
    const int ns = ke - kb;
    const int nb = ns + MS - 1;   // bundles this chunk consumes
    // hoisted-addressing path (3-D nests, one point per thread column); 2-D row
    // strips are DRAM-bound already and keep the generic path (smaller code)
    constexpr bool FAST = RX == 1 && NS::NLOOP == 3;
    using FS = FastState<NS, T, P, MS>;
    // planes of the ring the FAST path reads after the queue prologue: bundle
    // s + MS - SS is the oldest step s needs (SS == MS without a queue)
    constexpr int SS = FAST ? FS::smem_span(FORM) : MS;

    if (tid == 0) {
        for (int s = 0; s <= D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        if constexpr (P::static_tx() > 0) {
            mbar_expect_tx(&bars[D], P::static_tx());
            march_issue<P, NS, 0>(nullptr, maps, &bars[D], 0, orgx + maps.adjx, orgy, true, stat);
        }
        for (int B = 0; B < (FAST ? D : D - 1) && B < nb; ++B) {
            mbar_expect_tx(&bars[B % D], P::slot_tx());
            march_issue<P, NS, 0>(ring + (B % D) * P::slot_bytes(), maps, &bars[B % D], kb + B - (MS - 1), orgx + maps.adjx,
                                  orgy, false, stat);
        }
    }
    if constexpr (P::static_tx() > 0) mbar_wait(&bars[D], 0);
    // TMA transfers complete in any order: step 0 needs bundles 0 .. MS-1, the
    // loop below waits only for the newest bundle of each step (the FAST path
    // waits for them one by one in its queue prologue)
    if constexpr (!FAST)
        for (int B = 0; B < MS - 1 && B < nb; ++B) mbar_wait(&bars[B % D], 0);

    int pt[NS::NLOOP];
    M m{NaiveMem<NS, T, false>{args, pt}, ring, stat, 0, tx, ty, 0, orgx, orgy, {}};
    bool aligned = true;
#pragma unroll
    for (int a = 0; a < NS::NARR; ++a) {
        m.sh[a] = xshift<P, NS>(a, orgx + maps.adjx);
        if (P::staged(a) && m.sh[a] != 0) aligned = false;
    }
    using WP = WinPlan<NS, T, LAYOUT, TX, TY, BY, FORM, RX>;
    bool vec_ok = false;
    if constexpr (WP::usable()) {
        vec_ok = true;   // sharded: per plane below (planes that forward to a neighbour store scalars)
#pragma unroll
        for (int r = 0; r < NS::NSROW; ++r) {
            if (!WP::srow_on(r)) continue;
            const int a = NS::srow_arr(r);
            // the point group's first element must be 16-byte aligned
            if ((reinterpret_cast<uintptr_t>(args.arr[a].base) + (uintptr_t)orgx * sizeof(T)) % 16 != 0) vec_ok = false;
            for (int p = 0; p < NS::ndim(a); ++p) {
                const long long st = args.arr[a].stride[p];
                if (p == WP::sxpos(a) ? st != 1 : st % WP::V != 0) vec_ok = false;
            }
        }
    }

    T win[WP::usable() ? WP::total() : 1];   // register windows, carried across steps (queue)
    // RX == 1: the thread's per-array box offsets, global pointers and in-domain points (march-invariant)
    constexpr int NPX = TX / BX, NPY = TY / BY, NPTS = NPX * NPY;
    FS fs;
    unsigned toff[NS::NARR];
    bool inb[NPTS];
    T q[NS::NARR][NPTS][MS > 0 ? MS : 1];          // k-column queues (queued arrays only; the rest is dead)
    const int ly0 = ty * NPY;                       // the thread's first row (rows ly0 .. ly0 + NPY - 1)
    auto set_planes = [&](int newest) {
#pragma unroll
        for (int a = 0; a < NS::NARR; ++a) {
            if (!P::on_ring(a)) continue;
            const int mp = P::march_pos(a);
#pragma unroll
            for (int i = 0; i < MS; ++i) {
                if (i >= P::span(a)) continue;
                int slot = newest + D + NS::ld_lo(a, mp) + i - NS::ld_hi(a, mp);
                slot = slot >= D ? slot - D : slot;
                fs.plane[a][i] = (unsigned)(slot * P::slot_bytes() + P::ring_off(a)) + toff[a];
            }
        }
    };
    if constexpr (FAST) {
#pragma unroll
        for (int a = 0; a < NS::NARR; ++a) {
            toff[a] = 0;
            fs.gp[a] = nullptr;
            fs.gstep[a] = 0;
            if (P::staged(a)) {
                int e = 0;
#pragma unroll
                for (int p = 0; p < NS::ndim(a); ++p) {
                    const int sg = NS::ld_sig(a, p);
                    if (sg == P::X) e += (tx + m.sh[a] - P::lo(a, p)) * P::bstride(a, p);
                    else if (sg == P::Y) e += (ly0 - P::lo(a, p)) * P::bstride(a, p);
                }
                toff[a] = (unsigned)(e * (int)P::esize(a));
                if (P::is_static(a)) fs.stat[a] = (unsigned)(stat - ring) + (unsigned)P::static_off(a) + toff[a];
            }
            if (FS::needs_gp(a, FORM)) {
                long long e = 0, st = 0;
#pragma unroll
                for (int p = 0; p < NS::ndim(a); ++p) {
                    const int sg = NS::sig(a, p);
                    const long long sd = args.arr[a].stride[p];
                    if (sg == 0) {
                        e += (long long)kb * sd;
                        st += sd;
                    } else if (sg == P::X) e += (long long)(orgx + tx) * sd;
                    else if (NS::NLOOP == 3 && sg == 1) e += (long long)(orgy + ly0) * sd;
                }
                const int es = NS::is_int(a) ? 4 : (int)sizeof(T);
                fs.gp[a] = static_cast<char*>(args.arr[a].base) + e * es;
                fs.gstep[a] = st * es;
            }
        }
#pragma unroll
        for (int ry = 0; ry < NPY; ++ry)
#pragma unroll
            for (int rx = 0; rx < NPX; ++rx) {
                const int x = orgx + tx + rx * BX, y = orgy + ly0 + ry;
                inb[ry * NPX + rx] = x < args.hi[P::X] && x >= xlo0 && (NS::NLOOP < 3 || y < args.hi[1]);
            }
        if (ns > 0) {
            // queue prologue, bundle by bundle: the lower column planes of step 0
            // go to registers; a bundle no step reads from shared memory
            // (b < MS - SS) frees its slot for the bundle D further on
            set_planes((MS - 1) % D);
            for (int b = 0; b < MS - 1; ++b) {
                mbar_wait(&bars[b % D], (uint32_t)((b / D) & 1));
                fast_queue_fill<NS, P, FS, FORM, NPX, NPY, BX, 0, T>(ring, fs, q, b);
                if (b < MS - SS) {
                    __syncthreads();
                    if (tid == 0 && b + D < nb) {
                        fence_proxy_async();
                        mbar_expect_tx(&bars[b % D], P::slot_tx());
                        march_issue<P, NS, 0>(ring + (b % D) * P::slot_bytes(), maps, &bars[b % D],
                                              kb + b + D - (MS - 1), orgx + maps.adjx, orgy, false, stat);
                    }
                }
            }
        }
    }
    if constexpr (FAST) {
        // ring bookkeeping carried across steps (no division per step).  Step s
        // (s >= 1) frees bundle s-1+MS-SS (the oldest step s-1 read) and
        // issues bundle s-1+MS-SS+D into its slot; step 0's were issued above.
        int newest = (MS - 1) % D, phase = ((MS - 1) / D) & 1, islot = (MS - SS) % D;
        int ib = MS - SS + D;                       // next bundle to issue
        auto step = [&](int s) __attribute__((always_inline)) {
            __syncthreads();   // every thread is done with step s-1: its oldest slot is free
            if (s > 0) {
                if (tid == 0 && ib < nb) {
                    fence_proxy_async();
                    mbar_expect_tx(&bars[islot], P::slot_tx());
                    march_issue<P, NS, 0>(ring + islot * P::slot_bytes(), maps, &bars[islot], kb + ib - (MS - 1),
                                          orgx + maps.adjx, orgy, false, stat);
                }
                ++ib;
                islot = islot + 1 == D ? 0 : islot + 1;
            }
            mbar_wait(&bars[newest], (uint32_t)phase);
            pt[0] = kb + s;
            m.k = kb + s;
            m.newest = newest;
            // this step's ring planes: one add per (array, plane) for all of the thread's points
            set_planes(newest);
            fast_points<NS, P, M, FS, FORM, NPX, NPY, BX, 0>(m, fs, q, args, pt, inb, orgx + tx, orgy + ly0, tx, ly0);
            fast_queue_shift<NS, P, FS, FORM, NPTS, 0>(q);
#pragma unroll
            for (int a = 0; a < NS::NARR; ++a)
                if (FS::needs_gp(a, FORM)) fs.gp[a] += fs.gstep[a];
            if (++newest == D) {
                newest = 0;
                phase ^= 1;
            }
        };
        // unrolled by the march span: the k-column queue shifts become register renames
        constexpr int U = MS > 1 ? MS : 1;
        int s = 0;
        for (; s + U <= ns; s += U) {
#pragma unroll
            for (int u = 0; u < U; ++u) step(s + u);
        }
        for (; s < ns; ++s) step(s);
    } else {
    for (int s = 0; s < ns; ++s) {
        __syncthreads();   // every thread is done with step s-1: its oldest slot is free
        if (tid == 0) {
            const int B = s + D - 1;
            if (B < nb) {
                fence_proxy_async();
                mbar_expect_tx(&bars[B % D], P::slot_tx());
                march_issue<P, NS, 0>(ring + (B % D) * P::slot_bytes(), maps, &bars[B % D], kb + B - (MS - 1),
                                      orgx + maps.adjx, orgy, false, stat);
            }
        }
        const int Bw = s + MS - 1;
        mbar_wait(&bars[Bw % D], (uint32_t)((Bw / D) & 1));
        pt[0] = kb + s;
        m.k = kb + s;
        m.newest = Bw % D;
        if constexpr (WP::usable()) {
            if (aligned) {
                win_load<WP, M, NS, 0>(m, win, tx * RX, ty * WP::NY, s == 0);
                win_rows<WP, M, NS, FORM, 0, RX>(m, win, vec_ok, args, pt, tx * RX, ty * WP::NY, xlo0, orgy);
                win_shift<WP, T, 0>(win);
                continue;
            }
        }
        {
#pragma unroll
            for (int ry = 0; ry < TY / BY; ++ry) {
#pragma unroll
                for (int rx = 0; rx < TX / BX; ++rx) {
                    m.lx = RX > 1 ? tx * RX + rx : tx + rx * BX;
                    m.ly = ty + ry * BY;
                    const int x = orgx + m.lx, y = orgy + m.ly;
                    if (x < args.hi[P::X] && x >= xlo0 && (NS::NLOOP < 3 || y < args.hi[1])) {
                        pt[P::X] = x;
                        if constexpr (NS::NLOOP == 3) pt[1] = y;
                        NS::template body<FORM>(m, args.s, pt);
                    }
                }
            }
        }
    }
    }
    if (args.sh.enabled) __threadfence_system();   // peer write-through visible before the step flag
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

template <class NS, class T, int LAYOUT, int TX, int TY, int RX = 1>
bool encode_maps(const LaunchReq& r, TmaMaps<NS>& maps) {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY, RX>;
    EncodeTiledFn enc = tma_encoder();
    bool first_staged = true;
    maps.evict = 0;
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
        const int mis = (int)(reinterpret_cast<uintptr_t>(d->data) % 16);
        if (mis % es != 0) ACS_TMA_FAIL("base not element aligned");
        const int adj = mis / es;
        if (adj && !P::inner_is_x(a)) ACS_TMA_FAIL("unaligned base of an array whose innermost subscript is not x");
        // one shared shift: the kernel works in tensor-map x coordinates (x + adjx)
        if (first_staged) maps.adjx = adj;
        else if (maps.adjx != adj) ACS_TMA_FAIL("staged arrays with different base shifts");
        {
            static const bool ev = [] {
                const char* e = std::getenv("ACS_TMA_EVICT");
                return e && e[0] == '1';
            }();
            bool once = P::on_ring(a) && P::span(a) == 1;
            for (int p = 0; p < NS::ndim(a); ++p)
                if (NS::ld_sig(a, p) > 0 && (NS::ld_lo(a, p) != 0 || NS::ld_hi(a, p) != 0)) once = false;
            if (ev && once) maps.evict |= 1u << a;
        }
        first_staged = false;
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
            gdim[dd] = (cuuint64_t)(d->dims[p] + (dd == 0 ? adj : 0));
            box[dd] = (cuuint32_t)P::extent(a, p);
            estr[dd] = 1;
        }
        const CUtensorMapDataType dt = NS::is_int(a) ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                       : sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                        : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        void* base = static_cast<char*>(d->data) - (size_t)adj * es;
        CUresult e = enc(&maps.m[a], dt, (cuuint32_t)nd, base, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
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

template <class NS, class T, int FORM, int LAYOUT, int TX, int TY, int BX, int BY, int PF, int RX = 1, int KCH = 0>
acs_status launch_march(const LaunchReq& r) {
    using P = MarchPlan<NS, T, LAYOUT, TX, TY, RX>;
    static_assert(P::usable(), "march skeleton: nest not stageable");
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    TmaMaps<NS> maps;
    std::memset(&maps, 0, sizeof maps);
    if (!encode_maps<NS, T, LAYOUT, TX, TY, RX>(r, maps)) {
        // layout the TMA cannot describe (unaligned base / pitch): an explicit
        // slot request fails loudly; the DEFAULT schedule keeps the same
        // numerics through the global-memory skeleton
        if (r.strict) {
            set_error(std::string("march skeleton (") + NS::array_names[0] + ", ...) cannot describe this layout with the TMA "
                      "(16-byte aligned base and pitches needed); use the naive slot or native strides");
            return ACS_E_LAYOUT;
        }
        return launch_naive<NS, T, FORM>(r);
    }
    constexpr int D = march_ring_depth<NS, T, LAYOUT, TX, TY, RX, PF, FORM>();
    constexpr int smem = D * P::slot_bytes() + P::static_bytes() + (D + 1) * 8;
    auto kern = march_kernel<NS, T, FORM, LAYOUT, TX, TY, BX, BY, PF, RX>;
    static std::atomic<unsigned long long> attr_done{0};
    set_smem_attr_once(kern, smem, attr_done);
    constexpr int NL = NS::NLOOP;
    const long long xlo0 = ka.lo[NL - 1];
    const long long nx = ka.hi[NL - 1] - (P::ALIGNED ? xlo0 - ((((xlo0 + maps.adjx) % P::V) + P::V) % P::V) : xlo0);
    const long long ny = NL == 3 ? ka.hi[1] - ka.lo[1] : 1;
    const long long nz = ka.hi[0] - ka.lo[0];
    const long long tiles = ((nx + TX - 1) / TX) * (NL == 3 ? (ny + TY - 1) / TY : 1);
    // ~8 waves of CTAs; chunks long enough to amortise the (span-1)-plane prologue
    const long long want = (148LL * 4 * 8 + tiles - 1) / tiles;
    long long kchunk = (nz + want - 1) / want;
    const long long minch = 4LL * (P::maxspan() > 1 ? P::maxspan() : 2);
    // 2-D row strips: the shortest chunk the prologue allows (measured, tools/gpu/kchunk_sweep.sh:
    // calc2 6381 -> 6988 GB/s, pdv 6572 -> 6806 against ~100-row chunks); 3-D keeps ~8 waves
    if (NL == 2 || kchunk < minch) kchunk = minch;
    static const long long kch_env = [] {   // experiment knob (tools/gpu), not a tuning path
        const char* e = std::getenv("ACS_MARCH_KCHUNK");
        return e ? std::atoll(e) : 0LL;
    }();
    if (KCH > 0) kchunk = KCH;                // registered one-wave configurations
    else if (kch_env > 0) kchunk = kch_env;
    if (kchunk > nz) kchunk = nz;
    const long long chunks = (nz + kchunk - 1) / kchunk;
    dim3 grid((unsigned)((nx + TX - 1) / TX), (unsigned)(NL == 3 ? (ny + TY - 1) / TY : 1), (unsigned)chunks);
    if (r.preload) return preload_fn((const void*)kern);
    kern<<<grid, dim3(BX, BY, 1), smem, r.stream>>>(ka, maps, (int)kchunk);
    return check_launch("march");
}

template <class NS, class T, int LAYOUT, int TX, int TY, int BX, int BY, int PF, int RX = 1, int KCH = 0>
void fill_march(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_march<NS, T, 0, LAYOUT, TX, TY, BX, BY, PF, RX, KCH>;
    e.launch[prec][1][slot] = &launch_march<NS, T, 1, LAYOUT, TX, TY, BX, BY, PF, RX, KCH>;
    e.launch[prec][2][slot] = &launch_march<NS, T, 2, LAYOUT, TX, TY, BX, BY, PF, RX, KCH>;
    e.launch[prec][3][slot] = &launch_march<NS, T, 3, LAYOUT, TX, TY, BX, BY, PF, RX, KCH>;
    e.launch[prec][4][slot] = &launch_march<NS, T, 4, LAYOUT, TX, TY, BX, BY, PF, RX, KCH>;
    e.sched_name[prec][slot] = "march tile " + std::to_string(TX) + "x" + std::to_string(TY) + " block " +
                               std::to_string(BX) + "x" + std::to_string(BY) + " pf " + std::to_string(PF) +
                               (RX > 1 ? " regwin " + std::to_string(RX) : "") +
                               (KCH > 0 ? " k-chunk " + std::to_string(KCH) : "");
    for (int v = 0; v < 5; ++v)
        if (e.best[prec][v] == 0 && v != ACS_ORIGINAL) e.best[prec][v] = slot;
}

// Default skeleton set of a nest registered at run time (paper_2306_13002_b200/
// jit.py): naive, and the TMA march skeleton when the nest's loads are stageable.
template <class NS, class T>
void fill_default(Entry& e) {
    fill_naive<NS, T>(e, 0);
    if constexpr (NS::NLOOP == 3) {
        if constexpr (MarchPlan<NS, T, 0, 128, 4, 1>::usable()) fill_march<NS, T, 0, 128, 4, 128, 2, 3>(e, 0);
    } else if constexpr (NS::NLOOP == 2) {
        fill_naive_multi<NS, T, 2>(e, 0);
        if constexpr (MarchPlan<NS, T, 0, 128, 1, 1>::usable()) fill_march<NS, T, 0, 128, 1, 128, 1, 3>(e, 0);
    }
}

}  // namespace acs
