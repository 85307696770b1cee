// registry.hpp — host-side kernel registration (the backend's analogue of the
// reference's region registry: find_regions keys, proj/src/ast.cpp:390-398)
// and the generic launcher that binds acs_array / acs_scalar descriptors to a
// generated nest struct (csrc/gen/<nest>.cuh).
#pragma once

#include <array>
#include <atomic>
#include <cstdlib>

#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/accsat_b200.h"
#include "acs_device.cuh"

namespace acs {

void set_error(const std::string& msg);

struct LaunchReq {
    const acs_array* arrays;
    int n_arrays;
    const acs_scalar* scalars;
    int n_scalars;
    cudaStream_t stream;
    const acs_shard* shard = nullptr;   // slab-sharded launch (acs_launch_sharded)
    bool strict = false;   // explicit slot: a skeleton that cannot take the layout fails (ACS_E_LAYOUT)
    bool preload = false;  // load the kernel's code (acs_preload) instead of launching it
};

// CUDA lazy loading loads a kernel's code at its first launch and may wait for
// the device to drain first: a kernel first launched while another stream's
// acs_wait_ctr spins on a neighbour would deadlock.  acs_preload loads every
// skeleton of a kernel up front.
inline acs_status preload_fn(const void* kern) {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, kern) == cudaSuccess ? ACS_OK : ACS_E_CUDA;
}

using LaunchFn = acs_status (*)(const LaunchReq&);

// One registered region.  launch[precision][variant][slot]; precision 0 = the
// nest's declared type (double), 1 = the fp32 instantiation (wave4); slot 0 =
// the naive skeleton, slots 1.. = tiled (march) configurations.
constexpr int kMaxSched = 8;
struct Entry {
    std::string kernel_id, function;
    int region = 0;
    int n_loops = 0;
    std::vector<std::string> arrays, scalars;
    std::vector<int> scalar_is_int;
    int static_loads[5] = {0, 0, 0, 0, 0};
    int fma_count[5] = {0, 0, 0, 0, 0};
    LaunchFn launch[2][6][kMaxSched] = {};   // variant 5 = ACS_ORIGINAL_NVCC (naive slot only)
    LaunchFn tb2[2][5] = {};                 // two time steps per launch (kernels/tblock.cuh), ping-pong nests
    std::string tb2_name[2];
    int tb2_read = -1;                       // registry index of the array a tb2 step reads
    std::string sched_name[2][kMaxSched];
    int n_sched[2] = {1, 1};     // slot 0 (naive) always present once registered
    int best[2][6] = {};         // preferred slot per (precision, variant); acs_tune updates it
    bool soa_last_dim = false;   // backend layout: trailing component subscript made slowest (D3Q19 q)
    int inner_lo = -999;         // the innermost loop's constant lower bound (native row offset)
    bool row_offset = false;     // native layout: shift real arrays so interior rows are sector-aligned
                                 // (entries whose fast skeletons do not use the TMA)
    std::vector<int> component_last;  // per array: trailing subscript is an absolute component index
    struct Reach {
        int sliced, loaded, stored, ld_lo, ld_hi, st_lo, st_hi;
    };
    std::vector<Reach> reach;          // subscript-0 reach per array (acs_kernel_array_reach)
    // per array: unconditional static store targets of every form, one offset
    // (loop-mapped position) or constant (absolute position) per subscript
    std::vector<std::vector<std::array<int, 8>>> must_write;
    std::vector<std::array<int, 8>> loop_of;   // per array/position: loop index (NS::sig) or -1
    // iteration space of the marked loops for these scalars (half-open)
    acs_status (*space)(const acs_scalar* sc, int n, long long* lo, long long* hi) = nullptr;
};

void register_entry(Entry* e);
Entry* find_entry(const std::string& id);

inline acs_dtype real_dtype(bool f32) { return f32 ? ACS_F32 : ACS_F64; }

// Opt a kernel into more than 48 KB of dynamic shared memory once per device
// (function attributes are per device; launches may come from several
// threads, hence the atomic bitmask).
template <class K>
inline void set_smem_attr_once(K kern, int smem, std::atomic<unsigned long long>& done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ULL << (dev & 63);
    if (!(done.load(std::memory_order_acquire) & bit)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        done.fetch_or(bit, std::memory_order_acq_rel);
    }
}

// Binds descriptors to KernelArgs<NS>, validating names, ranks, dtypes and
// the static subscript range of the iteration space (the interpreter's
// bounds check, proj/src/interp.cpp:10-22, done once per launch).
template <class NS, bool F32>
acs_status bind(const LaunchReq& r, KernelArgs<NS>& ka, bool& empty) {
    long long dims[NS::NARR][8];
    for (int a = 0; a < NS::NARR; ++a) {
        const acs_array* d = nullptr;
        for (int i = 0; i < r.n_arrays; ++i)
            if (r.arrays[i].name && std::strcmp(r.arrays[i].name, NS::array_names[a]) == 0) d = &r.arrays[i];
        if (!d) {
            set_error(std::string("missing array argument '") + NS::array_names[a] + "'");
            return ACS_E_ARG;
        }
        if (d->ndim != NS::ndim(a)) {
            set_error(std::string("array '") + NS::array_names[a] + "' has rank " + std::to_string(d->ndim) +
                      ", nest declares " + std::to_string(NS::ndim(a)));
            return ACS_E_SHAPE;
        }
        const acs_dtype want = NS::is_int(a) ? ACS_I32 : real_dtype(F32);
        if (d->dtype != want) {
            set_error(std::string("array '") + NS::array_names[a] + "' has dtype " + std::to_string(d->dtype) +
                      ", kernel expects " + std::to_string(want));
            return ACS_E_SHAPE;
        }
        if (!d->data) {
            set_error(std::string("array '") + NS::array_names[a] + "' has a null data pointer");
            return ACS_E_ARG;
        }
        bool rowmajor = true;
        for (int p = 0; p < d->ndim; ++p) {
            if (d->dims[p] <= 0) {
                set_error(std::string("array '") + NS::array_names[a] + "' has a non-positive dim");
                return ACS_E_SHAPE;
            }
            if (d->strides[p] != 0) rowmajor = false;
            dims[a][p] = d->dims[p];
        }
        ka.arr[a].base = static_cast<char*>(d->data);
        long long st = 1;
        for (int p = d->ndim - 1; p >= 0; --p) {
            ka.arr[a].stride[p] = rowmajor ? st : d->strides[p];
            st *= d->dims[p];
        }
        for (int p = d->ndim; p < 8; ++p) ka.arr[a].stride[p] = 0;
    }
    for (int s = 0; s < NS::NSCALAR; ++s) {
        const acs_scalar* d = nullptr;
        for (int i = 0; i < r.n_scalars; ++i)
            if (r.scalars[i].name && std::strcmp(r.scalars[i].name, NS::scalar_names[s]) == 0) d = &r.scalars[i];
        if (!d) {
            set_error(std::string("missing scalar argument '") + NS::scalar_names[s] + "'");
            return ACS_E_ARG;
        }
        const long long iv = d->is_int ? d->i : (long long)d->d;
        const double dv = d->is_int ? (double)d->i : d->d;
        NS::set_scalar(ka.s, s, iv, dv);
    }
    std::memset(&ka.sh, 0, sizeof ka.sh);
    if (r.shard) {
        const acs_shard& sd = *r.shard;
        ka.sh.enabled = 1;
        ka.sh.origin = sd.origin;
        ka.sh.lo_thr = sd.own_lo + sd.halo;
        ka.sh.hi_thr = sd.own_hi - sd.halo;
        // never forward below the upper neighbour's first buffer plane (a slab
        // whose stores reach past its owned range but whose reads do not look
        // back, e.g. swim's j+1 stores with no j-1 halo)
        if (sd.hi_origin > ka.sh.hi_thr) ka.sh.hi_thr = sd.hi_origin;
        for (int i = 0; i < sd.n_sharded; ++i) {
            int a = -1;
            for (int b = 0; b < NS::NARR; ++b)
                if (sd.names[i] && std::strcmp(sd.names[i], NS::array_names[b]) == 0) a = b;
            if (a < 0) {
                set_error(std::string("shard: unknown array '") + (sd.names[i] ? sd.names[i] : "") + "'");
                return ACS_E_ARG;
            }
            if (NS::sig(a, 0) != 0 && NS::sig(a, 0) != -1) {
                set_error(std::string("shard: array '") + NS::array_names[a] + "' is not sliced along the outer loop");
                return ACS_E_ARG;
            }
            ka.sh.peer_lo[a] = static_cast<char*>(sd.lo_data[i]);
            ka.sh.peer_hi[a] = static_cast<char*>(sd.hi_data[i]);
            ka.sh.dlo[a] = (sd.origin - sd.lo_origin) * ka.arr[a].stride[0];
            ka.sh.dhi[a] = (sd.origin - sd.hi_origin) * ka.arr[a].stride[0];
        }
        // a slab without neighbours (one rank) runs exactly like a plain launch
        bool any = false;
        for (int a = 0; a < NS::NARR; ++a) any = any || ka.sh.peer_lo[a] || ka.sh.peer_hi[a];
        if (!any) ka.sh.enabled = 0;
    }
    long long lo[NS::NLOOP], hi[NS::NLOOP];
    NS::bounds(ka.s, lo, hi);
    empty = false;
    for (int l = 0; l < NS::NLOOP; ++l) {
        if (hi[l] <= lo[l]) empty = true;
        ka.lo[l] = (int)lo[l];
        ka.hi[l] = (int)hi[l];
    }
    if (empty) return ACS_OK;
    for (int a = 0; a < NS::NARR; ++a)
        for (int p = 0; p < NS::ndim(a); ++p) {
            const int sg = NS::sig(a, p);
            const long long mn = (sg >= 0 ? lo[sg] : 0) + NS::off_lo[a][p];
            const long long mx = (sg >= 0 ? hi[sg] - 1 : 0) + NS::off_hi[a][p];
            if (mn < 0 || mx >= dims[a][p]) {
                set_error(std::string("iteration space indexes '") + NS::array_names[a] + "' subscript " +
                          std::to_string(p) + " in [" + std::to_string(mn) + ", " + std::to_string(mx) +
                          "], outside [0, " + std::to_string(dims[a][p]) + ")");
                return ACS_E_BOUNDS;
            }
        }
    return ACS_OK;
}

inline acs_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return ACS_E_CUDA;
    }
    return ACS_OK;
}

template <class NS, class T, int FORM, int MINB = 1>
acs_status launch_naive(const LaunchReq& r) {
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    constexpr int NL = NS::NLOOP;
    dim3 block, grid;
    const long long nx = ka.hi[NL - 1] - ka.lo[NL - 1];
    if (NL == 1) {
        block = dim3(256, 1, 1);
        grid = dim3((unsigned)((nx + 255) / 256), 1, 1);
    } else {
        // a CTA covers whole rows of the innermost loop when they fit (256):
        // row-shifted stores (D3Q19 pushes) then share a 32-byte sector only
        // with stores of the same CTA (fewer partial-sector read-modify-writes)
        static const unsigned bx_env = [] {
            const char* e = std::getenv("ACS_NAIVE_BX");
            return e ? (unsigned)std::atoi(e) : 0u;
        }();
        const unsigned bx = bx_env && nx >= (long long)bx_env ? bx_env : (nx >= 256 ? 256 : nx >= 128 ? 128 : 32);
        const unsigned by = 256 / bx;
        const long long ny = ka.hi[NL - 2] - ka.lo[NL - 2];
        block = dim3(bx, by, 1);
        grid = dim3((unsigned)((nx + bx - 1) / bx), (unsigned)((ny + by - 1) / by),
                    NL >= 3 ? (unsigned)(ka.hi[0] - ka.lo[0]) : 1u);
    }
    // ORIGINAL keeps every as-written load and store (ld_asis); the emitted
    // forms use ordinary (read-only-path where legal) accesses.
    if (r.preload) return preload_fn((const void*)naive_kernel<NS, T, FORM, FORM == ACS_ORIGINAL, MINB>);
    naive_kernel<NS, T, FORM, FORM == ACS_ORIGINAL, MINB><<<grid, block, 0, r.stream>>>(ka);
    return check_launch(NS::array_names[0]);
}

template <class NS, class T, int FORM, int R>
acs_status launch_naive_multi(const LaunchReq& r) {
    KernelArgs<NS> ka;
    bool empty = false;
    acs_status st = bind<NS, std::is_same<T, float>::value>(r, ka, empty);
    if (st != ACS_OK || empty) return st;
    constexpr int NL = NS::NLOOP;
    static_assert(NL >= 2, "naive_multi: 2-D / 3-D nests");
    const long long nx = ka.hi[NL - 1] - ka.lo[NL - 1];
    const unsigned bx = nx >= 128 * R ? 128 : 32;
    const unsigned by = 256 / bx;
    const long long ny = ka.hi[NL - 2] - ka.lo[NL - 2];
    dim3 block(bx, by, 1);
    dim3 grid((unsigned)((nx + (long long)bx * R - 1) / ((long long)bx * R)), (unsigned)((ny + by - 1) / by),
              NL >= 3 ? (unsigned)(ka.hi[0] - ka.lo[0]) : 1u);
    if (r.preload) return preload_fn((const void*)naive_multi_kernel<NS, T, FORM, R>);
    naive_multi_kernel<NS, T, FORM, R><<<grid, block, 0, r.stream>>>(ka);
    return check_launch(NS::array_names[0]);
}

// naive with R points per thread (ORIGINAL registered too for parity coverage:
// its as-written loads are ordered, so its R bodies do not overlap)
template <class NS, class T, int R>
void fill_naive_multi(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_naive_multi<NS, T, 0, R>;
    e.launch[prec][1][slot] = &launch_naive_multi<NS, T, 1, R>;
    e.launch[prec][2][slot] = &launch_naive_multi<NS, T, 2, R>;
    e.launch[prec][3][slot] = &launch_naive_multi<NS, T, 3, R>;
    e.launch[prec][4][slot] = &launch_naive_multi<NS, T, 4, R>;
    e.sched_name[prec][slot] = "naive, " + std::to_string(R) + " points per thread";
    for (int v = 1; v < 5; ++v)
        if (e.best[prec][v] == 0) e.best[prec][v] = slot;
}

template <class NS, class T>
void fill_naive(Entry& e, int prec) {
    e.launch[prec][0][0] = &launch_naive<NS, T, 0>;
    e.launch[prec][1][0] = &launch_naive<NS, T, 1>;
    e.launch[prec][2][0] = &launch_naive<NS, T, 2>;
    e.launch[prec][3][0] = &launch_naive<NS, T, 3>;
    e.launch[prec][4][0] = &launch_naive<NS, T, 4>;
    e.launch[prec][5][0] = &launch_naive<NS, T, 5>;
    e.sched_name[prec][0] = "naive (one thread per point, as-written loads for ORIGINAL)";
}

// Extra naive slot with an occupancy floor: __launch_bounds__(256, MINB) caps
// registers so MINB CTAs (8*MINB warps) fit per SM — more loads in flight
// for register-heavy point-local nests (D3Q19).
template <class NS, class T, int MINB>
void fill_naive_occ(Entry& e, int prec) {
    const int slot = e.n_sched[prec]++;
    e.launch[prec][0][slot] = &launch_naive<NS, T, 0, MINB>;
    e.launch[prec][1][slot] = &launch_naive<NS, T, 1, MINB>;
    e.launch[prec][2][slot] = &launch_naive<NS, T, 2, MINB>;
    e.launch[prec][3][slot] = &launch_naive<NS, T, 3, MINB>;
    e.launch[prec][4][slot] = &launch_naive<NS, T, 4, MINB>;
    e.sched_name[prec][slot] = "naive, >= " + std::to_string(MINB) + " CTAs/SM";
}

template <class NS>
acs_status eval_space(const acs_scalar* sc, int n, long long* lo, long long* hi) {
    typename NS::Scalars s{};
    for (int i = 0; i < NS::NSCALAR; ++i) {
        const acs_scalar* d = nullptr;
        for (int j = 0; j < n; ++j)
            if (sc[j].name && std::strcmp(sc[j].name, NS::scalar_names[i]) == 0) d = &sc[j];
        if (!d) {
            set_error(std::string("missing scalar argument '") + NS::scalar_names[i] + "'");
            return ACS_E_ARG;
        }
        NS::set_scalar(s, i, d->is_int ? d->i : (long long)d->d, d->is_int ? (double)d->i : d->d);
    }
    NS::bounds(s, lo, hi);
    return ACS_OK;
}

template <class NS>
void describe(Entry& e, const char* file, int region) {
    e.space = &eval_space<NS>;
    e.inner_lo = NS::inner_lo_const;
    e.region = region;
    e.n_loops = NS::NLOOP;
    for (int a = 0; a < NS::NARR; ++a) {
        e.arrays.push_back(NS::array_names[a]);
        e.component_last.push_back(NS::ndim(a) >= 2 && NS::sig(a, NS::ndim(a) - 1) == -1 ? 1 : 0);
        Entry::Reach rc{};
        rc.sliced = NS::ndim(a) >= 2 && NS::sig(a, 0) == 0;
        rc.loaded = NS::is_loaded(a);
        rc.stored = !NS::readonly(a);
        rc.ld_lo = NS::ld_lo(a, 0);
        rc.ld_hi = NS::ld_hi(a, 0);
        rc.st_lo = NS::off_lo[a][0];   // union of load and store offsets: a safe bound for stores
        rc.st_hi = NS::off_hi[a][0];
        e.reach.push_back(rc);
        std::array<int, 8> lo_of{};
        for (int p = 0; p < 8; ++p) lo_of[p] = p < NS::ndim(a) ? NS::sig(a, p) : -1;
        e.loop_of.push_back(lo_of);
        e.must_write.emplace_back();
        for (int t = 0; t < NS::n_must_write; ++t)
            if (NS::must_write_arr[t] == a) {
                std::array<int, 8> o{};
                for (int p = 0; p < 8; ++p) o[p] = NS::must_write_off[t][p];
                e.must_write.back().push_back(o);
            }
    }
    for (int s = 0; s < NS::NSCALAR; ++s) {
        e.scalars.push_back(NS::scalar_names[s]);
        e.scalar_is_int.push_back(NS::scalar_is_int[s] ? 1 : 0);
    }
    for (int v = 0; v < 5; ++v) {
        e.static_loads[v] = NS::static_loads[v];
        e.fma_count[v] = NS::fma_count[v];
    }
    (void)file;
}

}  // namespace acs
