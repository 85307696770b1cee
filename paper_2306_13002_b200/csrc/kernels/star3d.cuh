// star3d.cuh — the B200 skeleton for 3-D star stencils (jacobi7: radius 1,
// wave4: radius 2).  2.5-D blocking:
//
//   * a CTA owns a TY x TX tile of (j, i) columns and marches along k over a
//     chunk of planes (grid z = chunks), so each plane of the stencil array is
//     fetched from HBM once per tile instead of 2R+1 times;
//   * each thread keeps the 2R+1 values of its own column (k-R .. k+R) in a
//     REGISTER QUEUE and prefetches the next plane one iteration ahead (the
//     paper's "common loads held in registers", applied across iterations);
//   * the current plane sits in a shared-memory tile with an R-wide halo, so
//     the j/i neighbours are LDS hits, and the centre comes from the queue;
//   * every other array (up, vel2, un; Anext) is streamed straight from/to
//     HBM, coalesced along i.
//
// The per-point arithmetic is the generated body of the requested form
// (original / emitted), so the skeleton never changes the numerics.
#pragma once

#include "../acs_device.cuh"

namespace acs {

template <class NS>
struct StarInfo {
    static constexpr int star() {
        for (int a = 0; a < NS::NARR; ++a)
            for (int p = 0; p < NS::ndim(a); ++p)
                if (NS::off_lo[a][p] != 0 || NS::off_hi[a][p] != 0) return a;
        return -1;
    }
    static constexpr int radius() {
        int r = 0;
        constexpr int s = star();
        if (s < 0) return 0;
        for (int p = 0; p < NS::ndim(s); ++p) {
            r = NS::off_hi[s][p] > r ? NS::off_hi[s][p] : r;
            r = -NS::off_lo[s][p] > r ? -NS::off_lo[s][p] : r;
        }
        return r;
    }
    static constexpr bool only_one_star() {
        int n = 0;
        for (int a = 0; a < NS::NARR; ++a) {
            bool off = false;
            for (int p = 0; p < NS::ndim(a); ++p)
                if (NS::off_lo[a][p] != 0 || NS::off_hi[a][p] != 0) off = true;
            n += off;
        }
        return n == 1;
    }
};

template <class NS, class T, int TX, int TY>
struct StarMem {
    static constexpr int S = StarInfo<NS>::star();
    static constexpr int R = StarInfo<NS>::radius();
    static constexpr int PITCH = TX + 2 * R;
    NaiveMem<NS, T, false> g;
    const T* q;      // register queue, q[R + dk]
    const T* sc;     // shared tile at this thread's centre

    template <int ARR>
    using elem_t = typename NaiveMem<NS, T, false>::template elem_t<ARR>;

    template <int ARR, int... O>
    __device__ __forceinline__ elem_t<ARR> ld() const {
        if constexpr (ARR == S) {
            constexpr int o[3] = {O...};
            static_assert(sizeof...(O) == 3, "star array must be 3-D");
            if constexpr (o[0] != 0) {
                static_assert(o[1] == 0 && o[2] == 0, "off-axis k neighbour: not a star stencil");
                return q[R + o[0]];
            } else if constexpr (o[1] == 0 && o[2] == 0) {
                return q[R];
            } else {
                return sc[o[1] * PITCH + o[2]];
            }
        } else {
            return g.template ld<ARR, O...>();
        }
    }
    template <int ARR, class... I>
    __device__ __forceinline__ elem_t<ARR> ldx(I... idx) const { return g.template ldx<ARR>(idx...); }
    template <int ARR, int... O>
    __device__ __forceinline__ void st(elem_t<ARR> v) const { g.template st<ARR, O...>(v); }
    template <int ARR, class... A>
    __device__ __forceinline__ void stx(A... args) const { g.template stx<ARR>(args...); }
};

template <class NS, class T, int FORM, int TX, int TY>
__global__ void __launch_bounds__(TX* TY) star3d_kernel(const __grid_constant__ KernelArgs<NS> args, int kchunk,
                                                        int dim1, int dim2) {
    constexpr int S = StarInfo<NS>::star();
    constexpr int R = StarInfo<NS>::radius();
    constexpr int PITCH = TX + 2 * R;
    constexpr int Q = 2 * R + 1;
    static_assert(NS::NLOOP == 3 && S >= 0 && NS::sig(S, 0) == 0 && NS::sig(S, 1) == 1 && NS::sig(S, 2) == 2,
                  "star3d needs a [k][j][i] star array");
    __shared__ T tile[(TY + 2 * R) * PITCH];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int i0 = args.lo[2] + blockIdx.x * TX, j0 = args.lo[1] + blockIdx.y * TY;
    const int i = i0 + tx, j = j0 + ty;
    const int kb = args.lo[0] + blockIdx.z * kchunk;
    const int ke = min(kb + kchunk, args.hi[0]);
    const bool active = i < args.hi[2] && j < args.hi[1];
    const bool inarr = i < dim2 && j < dim1;

    const T* A = reinterpret_cast<const T*>(args.arr[S].base);
    const long long sk = args.arr[S].stride[0], sj = args.arr[S].stride[1], si = args.arr[S].stride[2];
    const long long col = (long long)j * sj + (long long)i * si;

    T q[Q];
#pragma unroll
    for (int d = 0; d < Q - 1; ++d) q[d + 1] = inarr ? __ldg(A + (long long)(kb - R + d) * sk + col) : T(0);
    T next = inarr ? __ldg(A + (long long)(kb + R) * sk + col) : T(0);

    // halo work list: R rows above/below (full pitch incl. corners), R columns left/right
    constexpr int NH = 2 * R * PITCH + 2 * R * TY;
    const int tid = ty * TX + tx;

    int pt[3] = {0, j, i};
    for (int k = kb; k < ke; ++k) {
#pragma unroll
        for (int d = 0; d < Q - 1; ++d) q[d] = q[d + 1];
        q[Q - 1] = next;
        if (k + 1 < ke && inarr) next = __ldg(A + (long long)(k + 1 + R) * sk + col);

        __syncthreads();  // previous plane fully consumed
        tile[(ty + R) * PITCH + tx + R] = q[R];
        const T* plane = A + (long long)k * sk;
        for (int h = tid; h < NH; h += TX * TY) {
            int r, c;
            if (h < 2 * R * PITCH) {
                const int row = h / PITCH;
                r = row < R ? row : TY + row;  // rows 0..R-1 and TY+R..TY+2R-1
                c = h % PITCH;
            } else {
                const int h2 = h - 2 * R * PITCH;
                const int row = h2 / (2 * R), cc = h2 % (2 * R);
                r = R + row;
                c = cc < R ? cc : TX + cc;
            }
            const int gj = j0 - R + r, gi = i0 - R + c;
            if (gj >= 0 && gi >= 0 && gj < dim1 && gi < dim2)
                tile[r * PITCH + c] = __ldg(plane + (long long)gj * sj + (long long)gi * si);
        }
        __syncthreads();
        if (active) {
            pt[0] = k;
            StarMem<NS, T, TX, TY> m{NaiveMem<NS, T, false>{args, pt}, q, &tile[(ty + R) * PITCH + tx + R]};
            NS::template body<FORM>(m, args.s, pt);
        }
    }
}

template <class NS, class T, int FORM>
acs_status launch_star3d(const LaunchReq& r) {
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    constexpr int TX = 32, TY = 8;
    constexpr int S = StarInfo<NS>::star();
    // array extents of the star array (for halo guards)
    long long dim1 = 0, dim2 = 0;
    for (int a = 0; a < r.n_arrays; ++a)
        if (std::strcmp(r.arrays[a].name, NS::array_names[S]) == 0) {
            dim1 = r.arrays[a].dims[1];
            dim2 = r.arrays[a].dims[2];
        }
    const long long nx = ka.hi[2] - ka.lo[2], ny = ka.hi[1] - ka.lo[1], nz = ka.hi[0] - ka.lo[0];
    const long long bxy = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
    // enough CTAs for ~16 waves of 148 SMs; chunks of >= 8 planes amortise the queue priming
    long long want_chunks = (148LL * 8 * 16 + bxy - 1) / bxy;
    long long kchunk = (nz + want_chunks - 1) / want_chunks;
    if (kchunk < 8) kchunk = 8;
    if (kchunk > nz) kchunk = nz;
    const long long chunks = (nz + kchunk - 1) / kchunk;
    dim3 grid((unsigned)((nx + TX - 1) / TX), (unsigned)((ny + TY - 1) / TY), (unsigned)chunks);
    star3d_kernel<NS, T, FORM, TX, TY><<<grid, dim3(TX, TY, 1), 0, r.stream>>>(ka, (int)kchunk, (int)dim1, (int)dim2);
    return check_launch("star3d");
}

template <class NS, class T>
void fill_star3d(Entry& e, int prec) {
    static_assert(StarInfo<NS>::only_one_star(), "star3d: exactly one array may carry stencil offsets");
    e.launch[prec][0][1] = &launch_star3d<NS, T, 0>;
    e.launch[prec][1][1] = &launch_star3d<NS, T, 1>;
    e.launch[prec][2][1] = &launch_star3d<NS, T, 2>;
    e.launch[prec][3][1] = &launch_star3d<NS, T, 3>;
    e.launch[prec][4][1] = &launch_star3d<NS, T, 4>;
}

}  // namespace acs
