// abi.cu — the C ABI (include/accsat_b200.h): registry, launch dispatch,
// error reporting and the device data utilities (seeded fills, strided copies).
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "registry.hpp"
#include "tma.cuh"

#include <algorithm>
#include <cstring>

namespace acs {

#ifdef ACS_JIT_REGISTRY
// a library built by paper_2306_13002_b200/jit.py for one user nest file:
// its generated registration unit defines register_jit()
void register_jit();
#else
void register_jacobi7();
void register_swim();
void register_clover();
void register_wave4();
void register_d3q19();
void register_zsolve();
#endif

namespace {
thread_local std::string g_err;
std::vector<Entry*>& registry() {
    static std::vector<Entry*> r;
    return r;
}
std::once_flag g_once;
void init_registry() {
    std::call_once(g_once, [] {
#ifdef ACS_JIT_REGISTRY
        register_jit();
#else
        register_jacobi7();
        register_swim();
        register_clover();
        register_wave4();
        register_d3q19();
        register_zsolve();
#endif
    });
}
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

EncodeTiledFn tma_encoder() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}
void register_entry(Entry* e) { registry().push_back(e); }
Entry* find_entry(const std::string& id) {
    for (Entry* e : registry())
        if (e->kernel_id == id) return e;
    return nullptr;
}

// ---- seeded fills: the device twin of nests.make_inputs ---------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t idx) {
    uint64_t z = seed + (idx + 1ULL) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct StridedDesc {
    int ndim;
    long long dims[8];
    long long stride[8];
};

__device__ __forceinline__ long long strided_offset(const StridedDesc& d, long long flat) {
    long long off = 0;
    for (int p = d.ndim - 1; p >= 0; --p) {
        const long long ip = flat % d.dims[p];
        flat /= d.dims[p];
        off += ip * d.stride[p];
    }
    return off;
}

template <class T>
__global__ void fill_kernel(T* base, StridedDesc d, long long n, int kind, uint64_t seed, double lo, double hi,
                            double p, long long off) {
    const double span = __dsub_rn(hi, lo);
    const double w[3] = {1.0 / 3.0, 1.0 / 18.0, 1.0 / 36.0};
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < n; f += (long long)gridDim.x * blockDim.x) {
        double v;
        if (kind == ACS_FILL_CONST) {
            v = lo;
        } else {
            const double u = (double)(splitmix64(seed, (uint64_t)(f + off)) >> 11) * 0x1.0p-53;
            if (kind == ACS_FILL_MASK) {
                v = u < p ? 1.0 : 0.0;
            } else {
                const double x = __dadd_rn(lo, __dmul_rn(span, u));
                if (kind == ACS_FILL_D3Q19) {
                    const int q = (int)((f + off) % 19);
                    v = __dmul_rn(w[q == 0 ? 0 : (q <= 6 ? 1 : 2)], __dadd_rn(1.0, x));
                } else {
                    v = x;
                }
            }
        }
        base[strided_offset(d, f)] = (T)v;
    }
}

template <>
__global__ void fill_kernel<float>(float* base, StridedDesc d, long long n, int kind, uint64_t seed, double lo,
                                   double hi, double p, long long off) {
    const double span = __dsub_rn(hi, lo);
    const double w[3] = {1.0 / 3.0, 1.0 / 18.0, 1.0 / 36.0};
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < n; f += (long long)gridDim.x * blockDim.x) {
        double v;
        if (kind == ACS_FILL_CONST) {
            v = lo;
        } else {
            const double u = (double)(splitmix64(seed, (uint64_t)(f + off)) >> 11) * 0x1.0p-53;
            const double x = __dadd_rn(lo, __dmul_rn(span, u));
            const int q = (int)((f + off) % 19);
            v = kind == ACS_FILL_MASK ? (u < p ? 1.0 : 0.0)
                : kind == ACS_FILL_D3Q19 ? __dmul_rn(w[q == 0 ? 0 : (q <= 6 ? 1 : 2)], __dadd_rn(1.0, x))
                : x;
        }
        base[strided_offset(d, f)] = __double2float_rn(v);
    }
}

template <class D, class S>
__global__ void copy_kernel(D* dst, StridedDesc dd, const S* src, StridedDesc sd, long long n) {
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < n; f += (long long)gridDim.x * blockDim.x)
        dst[strided_offset(dd, f)] = (D)src[strided_offset(sd, f)];
}

namespace {

bool make_desc(const acs_array* a, StridedDesc& d, long long& n) {
    if (!a || a->ndim < 1 || a->ndim > 8 || !a->data) return false;
    d.ndim = a->ndim;
    bool rowmajor = true;
    for (int p = 0; p < a->ndim; ++p) {
        if (a->dims[p] <= 0) return false;
        d.dims[p] = a->dims[p];
        if (a->strides[p] != 0) rowmajor = false;
    }
    long long st = 1;
    for (int p = a->ndim - 1; p >= 0; --p) {
        d.stride[p] = rowmajor ? st : a->strides[p];
        st *= a->dims[p];
    }
    n = st;
    return true;
}

int precision_of(const acs_array* arrays, int n) {
    for (int i = 0; i < n; ++i)
        if (arrays[i].dtype == ACS_F32) return 1;
    return 0;
}

int grid_for(long long n) {
    long long g = (n + 255) / 256;
    const long long cap = 148LL * 16;  // persistent-ish: 16 CTAs per SM, grid-stride
    return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

}  // namespace
}  // namespace acs

using namespace acs;

typedef CUresult (*GetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

static acs_status launch_impl(const acs_kernel* k, acs_variant variant, acs_schedule schedule, const acs_array* arrays,
                              int n_arrays, const acs_scalar* scalars, int n_scalars, const acs_shard* shard,
                              void* cuda_stream);

// stream-ordered cross-rank step flags (release / acquire at system scope)
__global__ void signal_kernel(unsigned long long* a, unsigned long long* b, unsigned long long v) {
    __threadfence_system();   // this stream's earlier kernels' stores (incl. peer stores) before the flag
    if (a) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
    if (b) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(b), "l"(v) : "memory");
}

__global__ void wait_kernel(const unsigned long long* a, const unsigned long long* b, unsigned long long v,
                            unsigned long long timeout_ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (const unsigned long long* f : {a, b}) {
        if (!f) continue;
        for (;;) {
            unsigned long long x;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
            if (x >= v) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) __trap();   // a peer never arrived: fail loudly
            __nanosleep(200);
        }
    }
    __threadfence_system();
}

// graph-capturable variants: the step value lives in a device counter, so one
// captured (wait, launch, signal) sequence replays for every step
__global__ void signal_ctr_kernel(unsigned long long* a, unsigned long long* b, unsigned long long* ctr) {
    __threadfence_system();
    const unsigned long long v = *ctr + 1;
    *ctr = v;
    if (a) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
    if (b) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(b), "l"(v) : "memory");
}

__global__ void wait_ctr_kernel(const unsigned long long* a, const unsigned long long* b,
                                const unsigned long long* ctr, unsigned long long timeout_ns) {
    const unsigned long long v = *ctr;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (const unsigned long long* f : {a, b}) {
        if (!f) continue;
        for (;;) {
            unsigned long long x;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
            if (x >= v) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) __trap();
            __nanosleep(200);
        }
    }
    __threadfence_system();
}

extern "C" {

int acs_abi_version(void) { return ACS_ABI_VERSION; }
const char* acs_last_error(void) { return g_err.c_str(); }

int acs_kernel_count(void) {
    init_registry();
    return (int)registry().size();
}

const char* acs_kernel_id(int index) {
    init_registry();
    if (index < 0 || index >= (int)registry().size()) return nullptr;
    return registry()[index]->kernel_id.c_str();
}

acs_status acs_lookup(const char* kernel_id, const acs_kernel** out) {
    init_registry();
    if (!kernel_id || !out) {
        set_error("acs_lookup: null argument");
        return ACS_E_ARG;
    }
    Entry* e = find_entry(kernel_id);
    if (!e) {
        set_error(std::string("no kernel registered for '") + kernel_id + "'");
        return ACS_E_NO_KERNEL;
    }
    *out = reinterpret_cast<const acs_kernel*>(e);
    return ACS_OK;
}

acs_status acs_kernel_get_info(const acs_kernel* k, acs_kernel_info* out) {
    if (!k || !out) {
        set_error("acs_kernel_get_info: null argument");
        return ACS_E_ARG;
    }
    const Entry* e = reinterpret_cast<const Entry*>(k);
    out->kernel_id = e->kernel_id.c_str();
    out->function = e->function.c_str();
    out->region = e->region;
    out->n_loops = e->n_loops;
    out->n_arrays = (int)e->arrays.size();
    out->n_scalars = (int)e->scalars.size();
    for (int v = 0; v < 5; ++v) {
        out->static_loads[v] = e->static_loads[v];
        out->fma_count[v] = e->fma_count[v];
    }
    out->has_tiled = e->n_sched[0] > 1;
    out->has_f32 = e->launch[1][0][0] != nullptr;
    out->n_schedules = e->n_sched[0];
    return ACS_OK;
}

const char* acs_kernel_array_name(const acs_kernel* k, int index) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || index < 0 || index >= (int)e->arrays.size()) return nullptr;
    return e->arrays[index].c_str();
}
acs_status acs_kernel_array_reach(const acs_kernel* k, int index, int* sliced, int* loaded, int* stored, int* ld_lo,
                                  int* ld_hi, int* st_lo, int* st_hi) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || index < 0 || index >= (int)e->reach.size() || !sliced || !loaded || !stored || !ld_lo || !ld_hi ||
        !st_lo || !st_hi) {
        set_error("acs_kernel_array_reach: bad argument");
        return ACS_E_ARG;
    }
    const Entry::Reach& r = e->reach[index];
    *sliced = r.sliced;
    *loaded = r.loaded;
    *stored = r.stored;
    *ld_lo = r.ld_lo;
    *ld_hi = r.ld_hi;
    *st_lo = r.st_lo;
    *st_hi = r.st_hi;
    return ACS_OK;
}

acs_status acs_kernel_must_write(const acs_kernel* k, int index, int32_t* loop_of, int max_targets, int32_t* offsets,
                                 int* n_targets) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || index < 0 || index >= (int)e->must_write.size() || !n_targets || max_targets < 0 ||
        (max_targets > 0 && !offsets)) {
        set_error("acs_kernel_must_write: bad argument");
        return ACS_E_ARG;
    }
    if (loop_of)
        for (int p = 0; p < ACS_MAX_DIMS; ++p) loop_of[p] = e->loop_of[index][p];
    const auto& t = e->must_write[index];
    *n_targets = (int)t.size();
    for (int i = 0; i < (int)t.size() && i < max_targets; ++i)
        for (int p = 0; p < ACS_MAX_DIMS; ++p) offsets[i * ACS_MAX_DIMS + p] = t[i][p];
    return ACS_OK;
}

acs_status acs_kernel_iteration_space(const acs_kernel* k, const acs_scalar* scalars, int n_scalars, int64_t* lo,
                                      int64_t* hi) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || !e->space || (n_scalars > 0 && !scalars) || !lo || !hi) {
        set_error("acs_kernel_iteration_space: bad argument");
        return ACS_E_ARG;
    }
    long long l[ACS_MAX_DIMS], h[ACS_MAX_DIMS];
    const acs_status st = e->space(scalars, n_scalars, l, h);
    if (st != ACS_OK) return st;
    for (int d = 0; d < e->n_loops; ++d) {
        lo[d] = l[d];
        hi[d] = h[d];
    }
    return ACS_OK;
}

acs_status acs_copy_box(void* dst, const void* src, int elem_size, int ndim, const int64_t* dims,
                        const int64_t* box_lo, const int64_t* box_hi, int kind, void* cuda_stream) {
    if (!dst || !src || elem_size <= 0 || ndim < 1 || ndim > ACS_MAX_DIMS || !dims || !box_lo || !box_hi ||
        kind < 0 || kind > 3) {
        set_error("acs_copy_box: bad argument");
        return ACS_E_ARG;
    }
    for (int p = 0; p < ndim; ++p) {
        if (dims[p] < 0 || box_lo[p] < 0 || box_hi[p] > dims[p]) {
            set_error("acs_copy_box: box outside the array");
            return ACS_E_BOUNDS;
        }
        if (box_hi[p] <= box_lo[p]) return ACS_OK;   // empty box
    }
    // innermost position k whose inner positions are all full: one contiguous run
    int k = ndim - 1;
    while (k > 0 && box_lo[k] == 0 && box_hi[k] == dims[k]) --k;
    size_t inner = (size_t)elem_size;   // bytes of one index step at position k
    for (int p = k + 1; p < ndim; ++p) inner *= (size_t)dims[p];
    const size_t width = inner * (size_t)(box_hi[k] - box_lo[k]);
    const size_t pitch = inner * (size_t)dims[k];
    const int64_t h_dim = k >= 1 ? dims[k - 1] : 1;
    const int64_t h_lo = k >= 1 ? box_lo[k - 1] : 0, h_n = k >= 1 ? box_hi[k - 1] - box_lo[k - 1] : 1;
    const int64_t d_lo = k >= 2 ? box_lo[k - 2] : 0, d_n = k >= 2 ? box_hi[k - 2] - box_lo[k - 2] : 1;
    const size_t slice = pitch * (size_t)h_dim;
    const size_t block = k >= 2 ? slice * (size_t)dims[k - 2] : slice;   // bytes of one step at position k-3
    static const cudaMemcpyKind kinds[4] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                                            cudaMemcpyDeviceToDevice, cudaMemcpyDefault};
    // positions outside k-2 are iterated here (row-major offset of the outer index)
    int64_t outer_n = 1;
    for (int p = 0; p < k - 2; ++p) outer_n *= box_hi[p] - box_lo[p];
    for (int64_t o = 0; o < outer_n; ++o) {
        size_t off = 0, rem = (size_t)o, mul = block;
        for (int p = k - 3; p >= 0; --p) {
            const int64_t n = box_hi[p] - box_lo[p];
            off += (size_t)(box_lo[p] + (int64_t)(rem % (size_t)n)) * mul;
            rem /= (size_t)n;
            mul *= (size_t)dims[p];
        }
        const size_t base = off + (size_t)d_lo * slice + (size_t)h_lo * pitch + (size_t)box_lo[k] * inner;
        cudaMemcpy3DParms prm = {};
        prm.srcPtr = make_cudaPitchedPtr(const_cast<char*>(static_cast<const char*>(src)) + base, pitch, width,
                                         (size_t)h_dim);
        prm.dstPtr = make_cudaPitchedPtr(static_cast<char*>(dst) + base, pitch, width, (size_t)h_dim);
        prm.extent = make_cudaExtent(width, (size_t)h_n, (size_t)d_n);
        prm.kind = kinds[kind];
        cudaError_t err = cudaMemcpy3DAsync(&prm, static_cast<cudaStream_t>(cuda_stream));
        if (err != cudaSuccess) {
            set_error(std::string("acs_copy_box: ") + cudaGetErrorString(err));
            return ACS_E_CUDA;
        }
    }
    return ACS_OK;
}

const char* acs_kernel_scalar_name(const acs_kernel* k, int index) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || index < 0 || index >= (int)e->scalars.size()) return nullptr;
    return e->scalars[index].c_str();
}
int acs_kernel_scalar_is_int(const acs_kernel* k, int index) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || index < 0 || index >= (int)e->scalars.size()) return -1;
    return e->scalar_is_int[index];
}

acs_status acs_launch(const acs_kernel* k, acs_variant variant, acs_schedule schedule, const acs_array* arrays,
                      int n_arrays, const acs_scalar* scalars, int n_scalars, void* cuda_stream) {
    return launch_impl(k, variant, schedule, arrays, n_arrays, scalars, n_scalars, nullptr, cuda_stream);
}

}  // extern "C"

static acs_status launch_impl(const acs_kernel* k, acs_variant variant, acs_schedule schedule, const acs_array* arrays,
                              int n_arrays, const acs_scalar* scalars, int n_scalars, const acs_shard* shard,
                              void* cuda_stream) {
    if (!k || (n_arrays > 0 && !arrays) || (n_scalars > 0 && !scalars)) {
        set_error("acs_launch: null argument");
        return ACS_E_ARG;
    }
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if ((int)variant < 0 || (int)variant > 5) {
        set_error("acs_launch: unknown variant");
        return ACS_E_ARG;
    }
    const int prec = precision_of(arrays, n_arrays);
    int slot;
    if (schedule == ACS_SCHED_DEFAULT)
        slot = (variant == ACS_ORIGINAL || variant == ACS_ORIGINAL_NVCC) ? 0 : e->best[prec][variant];
    else if (schedule == ACS_SCHED_NAIVE)
        slot = 0;
    else if (schedule == ACS_SCHED_TILED)
        slot = e->best[prec][variant] > 0 ? e->best[prec][variant] : 1;
    else
        slot = (int)schedule - 16;
    LaunchFn fn = (slot >= 0 && slot < kMaxSched) ? e->launch[prec][variant][slot] : nullptr;
    if (!fn) {
        set_error(e->kernel_id + ": no kernel in schedule slot " + std::to_string(slot) + " for variant " +
                  std::to_string(variant) + (prec ? " (fp32)" : ""));
        return ACS_E_NO_KERNEL;
    }
    LaunchReq r{arrays, n_arrays, scalars, n_scalars, static_cast<cudaStream_t>(cuda_stream), shard,
                (int)schedule >= 16};   // an explicit slot fails loudly on a layout it cannot take
    return fn(r);
}

extern "C" {

acs_status acs_launch_sharded(const acs_kernel* k, acs_variant variant, acs_schedule schedule, const acs_array* arrays,
                              int n_arrays, const acs_scalar* scalars, int n_scalars, const acs_shard* shard,
                              void* cuda_stream) {
    if (!shard || shard->n_sharded < 0 || shard->n_sharded > ACS_MAX_SHARDED || shard->own_hi < shard->own_lo ||
        shard->halo < 0) {
        set_error("acs_launch_sharded: bad shard descriptor");
        return ACS_E_ARG;
    }
    return launch_impl(k, variant, schedule, arrays, n_arrays, scalars, n_scalars, shard, cuda_stream);
}

acs_status acs_signal(uint64_t* flag_a, uint64_t* flag_b, uint64_t value, void* cuda_stream) {
    signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(cuda_stream)>>>((unsigned long long*)flag_a,
                                                                      (unsigned long long*)flag_b, value);
    return check_launch("acs_signal");
}

acs_status acs_wait(const uint64_t* flag_a, const uint64_t* flag_b, uint64_t value, int timeout_ms, void* cuda_stream) {
    wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(cuda_stream)>>>((const unsigned long long*)flag_a,
                                                                    (const unsigned long long*)flag_b, value,
                                                                    (unsigned long long)timeout_ms * 1000000ULL);
    return check_launch("acs_wait");
}

acs_status acs_launch_steps(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                            const acs_scalar* scalars, int n_scalars, int nsteps, int blocked, void* cuda_stream,
                            int* latest) {
    if (!k || !arrays || n_arrays != 2 || nsteps < 0 || !latest || (int)variant < 0 || (int)variant > 4) {
        set_error("acs_launch_steps: a ping-pong nest (two arrays), nsteps >= 0, a latest out-parameter");
        return ACS_E_ARG;
    }
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (e->arrays.size() != 2) {
        set_error(e->kernel_id + ": acs_launch_steps needs a two-array ping-pong nest");
        return ACS_E_ARG;
    }
    // the array each step reads (loaded, never stored) and the one it writes
    int rd = -1;
    for (int a = 0; a < 2; ++a)
        if (e->reach[a].loaded && !e->reach[a].stored) rd = a;
    if (rd < 0 || !e->reach[1 - rd].stored) {
        set_error(e->kernel_id + ": not a ping-pong nest (one array read, the other written)");
        return ACS_E_ARG;
    }
    int ir = -1, iw = -1;   // positions in `arrays`
    for (int i = 0; i < 2; ++i) {
        if (arrays[i].name && e->arrays[rd] == arrays[i].name) ir = i;
        if (arrays[i].name && e->arrays[1 - rd] == arrays[i].name) iw = i;
    }
    if (ir < 0 || iw < 0) {
        set_error(e->kernel_id + ": acs_launch_steps: arrays must be named " + e->arrays[0] + ", " + e->arrays[1]);
        return ACS_E_ARG;
    }
    const int prec = precision_of(arrays, n_arrays);
    acs_array cur = arrays[ir], oth = arrays[iw];
    const cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    int left = nsteps;
    while (left > 0) {
        acs_array step[2];
        step[ir] = cur;
        step[iw] = oth;
        step[ir].name = arrays[ir].name;
        step[iw].name = arrays[iw].name;
        acs_status st;
        LaunchFn tb = blocked ? e->tb2[prec][variant] : nullptr;
        if (tb && left >= 2) {
            LaunchReq r{step, 2, scalars, n_scalars, s};
            st = tb(r);
            left -= 2;
        } else {
            st = launch_impl(k, variant, ACS_SCHED_DEFAULT, step, 2, scalars, n_scalars, nullptr, cuda_stream);
            left -= 1;
        }
        if (st != ACS_OK) return st;
        std::swap(cur.data, oth.data);   // the written buffer is read next
    }
    *latest = cur.data == arrays[ir].data ? ir : iw;
    return ACS_OK;
}

acs_status acs_launch_leapfrog2(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                                const acs_scalar* scalars, int n_scalars, const acs_array* un2, void* cuda_stream) {
    if (!k || !arrays || n_arrays < 1 || !un2 || (int)variant < 0 || (int)variant > 4) {
        set_error("acs_launch_leapfrog2: the nest's arrays, a fourth buffer un2, a variant 0..4");
        return ACS_E_ARG;
    }
    const Entry* e = reinterpret_cast<const Entry*>(k);
    const int prec = precision_of(arrays, n_arrays);
    LaunchFn tb = e->tb2[prec][variant];
    if (!tb || e->arrays.size() != 4) {
        set_error(e->kernel_id + ": no two-step leapfrog kernel registered" + (prec ? " (fp32)" : " (fp64)"));
        return ACS_E_NO_KERNEL;
    }
    std::vector<acs_array> all(arrays, arrays + n_arrays);
    all.push_back(*un2);
    all.back().name = "un2";
    LaunchReq r{all.data(), (int)all.size(), scalars, n_scalars, static_cast<cudaStream_t>(cuda_stream)};
    return tb(r);
}

acs_status acs_eval_host(const acs_kernel* k, acs_variant variant, const acs_array* host, int n_arrays,
                         const acs_scalar* scalars, int n_scalars) {
    if (!k || (n_arrays > 0 && !host) || (n_scalars > 0 && !scalars)) {
        set_error("acs_eval_host: null argument");
        return ACS_E_ARG;
    }
    const Entry* e = reinterpret_cast<const Entry*>(k);
    static const int esize[5] = {8, 4, 4, 8, 1};
    std::vector<acs_array> dev(host, host + n_arrays);
    std::vector<void*> bufs((size_t)n_arrays, nullptr);
    std::vector<size_t> bytes((size_t)n_arrays, 0);
    auto fail = [&](const std::string& what, cudaError_t err) {
        for (void* b : bufs)
            if (b) cudaFree(b);
        set_error("acs_eval_host: " + what + ": " + cudaGetErrorString(err));
        return ACS_E_CUDA;
    };
    for (int i = 0; i < n_arrays; ++i) {
        const acs_array& a = host[i];
        if ((int)a.dtype < 0 || (int)a.dtype > 4 || a.ndim < 1 || a.ndim > ACS_MAX_DIMS || !a.data) {
            set_error(std::string("acs_eval_host: bad array '") + (a.name ? a.name : "") + "'");
            return ACS_E_ARG;
        }
        size_t n = 1;
        for (int p = 0; p < a.ndim; ++p) {
            if (a.strides[p] != 0) {
                set_error("acs_eval_host: host arrays are row-major (strides 0)");
                return ACS_E_ARG;
            }
            n *= (size_t)a.dims[p];
        }
        bytes[i] = n * (size_t)esize[a.dtype];
        cudaError_t err = cudaMalloc(&bufs[i], bytes[i] ? bytes[i] : 1);
        if (err != cudaSuccess) return fail("cudaMalloc", err);
        err = cudaMemcpy(bufs[i], a.data, bytes[i], cudaMemcpyHostToDevice);
        if (err != cudaSuccess) return fail("upload", err);
        dev[i].data = bufs[i];
    }
    acs_status st = launch_impl(k, variant, ACS_SCHED_DEFAULT, dev.data(), n_arrays, scalars, n_scalars, nullptr,
                                nullptr);
    cudaError_t err = cudaDeviceSynchronize();
    if (st == ACS_OK && err != cudaSuccess) return fail("launch", err);
    for (int i = 0; i < n_arrays && st == ACS_OK; ++i) {
        bool stored = true;   // unknown names: copy back (the post-state keeps every array)
        for (size_t a = 0; a < e->arrays.size(); ++a)
            if (host[i].name && e->arrays[a] == host[i].name) stored = e->reach[a].stored;
        if (!stored) continue;
        err = cudaMemcpy(host[i].data, bufs[i], bytes[i], cudaMemcpyDeviceToHost);
        if (err != cudaSuccess) return fail("download", err);
    }
    for (void* b : bufs)
        if (b) cudaFree(b);
    return st;
}

acs_status acs_preload(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                       const acs_scalar* scalars, int n_scalars) {
    if (!k || (int)variant < 0 || (int)variant > 5) {
        set_error("acs_preload: bad argument");
        return ACS_E_ARG;
    }
    const Entry* e = reinterpret_cast<const Entry*>(k);
    const int prec = precision_of(arrays, n_arrays);
    LaunchReq r{arrays, n_arrays, scalars, n_scalars, nullptr, nullptr, false, true};
    for (int slot = 0; slot < kMaxSched; ++slot) {
        LaunchFn fn = e->launch[prec][variant][slot];
        if (!fn) continue;
        const acs_status st = fn(r);
        if (st != ACS_OK && st != ACS_E_LAYOUT) return st;
    }
    // the step-ordering kernels too
    if (preload_fn((const void*)wait_ctr_kernel) != ACS_OK || preload_fn((const void*)signal_ctr_kernel) != ACS_OK) {
        set_error("acs_preload: cudaFuncGetAttributes failed");
        return ACS_E_CUDA;
    }
    return ACS_OK;
}

acs_status acs_signal_ctr(uint64_t* flag_a, uint64_t* flag_b, uint64_t* counter, void* cuda_stream) {
    if (!counter) {
        set_error("acs_signal_ctr: null counter");
        return ACS_E_ARG;
    }
    signal_ctr_kernel<<<1, 1, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
        (unsigned long long*)flag_a, (unsigned long long*)flag_b, (unsigned long long*)counter);
    return check_launch("acs_signal_ctr");
}

acs_status acs_wait_ctr(const uint64_t* flag_a, const uint64_t* flag_b, const uint64_t* counter, int timeout_ms,
                        void* cuda_stream) {
    if (!counter) {
        set_error("acs_wait_ctr: null counter");
        return ACS_E_ARG;
    }
    wait_ctr_kernel<<<1, 1, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
        (const unsigned long long*)flag_a, (const unsigned long long*)flag_b, (const unsigned long long*)counter,
        (unsigned long long)timeout_ms * 1000000ULL);
    return check_launch("acs_wait_ctr");
}

acs_status acs_ipc_export(const void* dptr, void* handle_out, int64_t* offset_out) {
    if (!dptr || !handle_out || !offset_out) {
        set_error("acs_ipc_export: null argument");
        return ACS_E_ARG;
    }
    static GetAddressRangeFn range = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (GetAddressRangeFn) nullptr;
        return reinterpret_cast<GetAddressRangeFn>(p);
    }();
    if (!range) {
        set_error("acs_ipc_export: cuMemGetAddressRange unavailable");
        return ACS_E_NCCL;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS) {
        set_error("acs_ipc_export: not a device allocation");
        return ACS_E_ARG;
    }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) {
        set_error(std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
        return ACS_E_CUDA;
    }
    std::memcpy(handle_out, &h, sizeof h);
    *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dptr) - base);
    return ACS_OK;
}

acs_status acs_ipc_import(const void* handle, int64_t offset, void** dptr_out) {
    if (!handle || !dptr_out) {
        set_error("acs_ipc_import: null argument");
        return ACS_E_ARG;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        set_error(std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        return ACS_E_CUDA;
    }
    *dptr_out = static_cast<char*>(base) + offset;
    return ACS_OK;
}

acs_status acs_ipc_close(void* dptr, int64_t offset) {
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(dptr) - offset);
    if (e != cudaSuccess) {
        set_error(std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
        return ACS_E_CUDA;
    }
    return ACS_OK;
}

const char* acs_kernel_schedule_name(const acs_kernel* k, int precision, int slot) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || precision < 0 || precision > 1 || slot < 0 || slot >= kMaxSched || !e->launch[precision][0][slot])
        return nullptr;
    return e->sched_name[precision][slot].c_str();
}

acs_status acs_tune(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                    const acs_scalar* scalars, int n_scalars, void* cuda_stream, int reps, int* best_slot,
                    float* ms_per_launch) {
    if (!k || (int)variant < 0 || (int)variant > 4 || reps < 1) {
        set_error("acs_tune: bad argument");
        return ACS_E_ARG;
    }
    Entry* e = const_cast<Entry*>(reinterpret_cast<const Entry*>(k));
    const int prec = precision_of(arrays, n_arrays);
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    LaunchReq r{arrays, n_arrays, scalars, n_scalars, s, nullptr, true};
    // candidates: every registered slot that takes this layout (one warm-up
    // launch each: TMA attributes, code loading)
    std::vector<int> cand;
    for (int slot = 0; slot < kMaxSched; ++slot) {
        if (ms_per_launch) ms_per_launch[slot] = -1.0f;
        LaunchFn fn = e->launch[prec][variant][slot];
        if (!fn) continue;
        const acs_status st = fn(r);
        if (st == ACS_E_LAYOUT) continue;   // this skeleton cannot take the layout: not a candidate
        if (st != ACS_OK) return st;
        cand.push_back(slot);
    }
    if (cand.empty()) {
        set_error("acs_tune: no registered schedule");
        return ACS_E_NO_KERNEL;
    }
    // repetitions interleaved across the candidates (a clock / power-cap drift
    // over the tuning run hits every slot alike), per-launch events, median
    const size_t nc = cand.size();
    std::vector<cudaEvent_t> ev(nc * (size_t)reps * 2);
    for (auto& x : ev) cudaEventCreate(&x);
    for (int i = 0; i < reps; ++i)
        for (size_t c = 0; c < nc; ++c) {
            cudaEventRecord(ev[(c * reps + i) * 2], s);
            e->launch[prec][variant][cand[c]](r);
            cudaEventRecord(ev[(c * reps + i) * 2 + 1], s);
        }
    if (cudaEventSynchronize(ev.back()) != cudaSuccess) {
        for (auto& x : ev) cudaEventDestroy(x);
        return check_launch("acs_tune");
    }
    float best = 1e30f;
    int bslot = -1;
    for (size_t c = 0; c < nc; ++c) {
        std::vector<float> t((size_t)reps);
        for (int i = 0; i < reps; ++i) cudaEventElapsedTime(&t[i], ev[(c * reps + i) * 2], ev[(c * reps + i) * 2 + 1]);
        std::sort(t.begin(), t.end());
        const float ms = reps % 2 ? t[reps / 2] : 0.5f * (t[reps / 2 - 1] + t[reps / 2]);
        if (ms_per_launch) ms_per_launch[cand[c]] = ms;
        if (ms < best) {
            best = ms;
            bslot = cand[c];
        }
    }
    for (auto& x : ev) cudaEventDestroy(x);
    if (bslot < 0) {
        set_error("acs_tune: no registered schedule");
        return ACS_E_NO_KERNEL;
    }
    e->best[prec][variant] = bslot;
    if (best_slot) *best_slot = bslot;
    return check_launch("acs_tune");
}

}  // extern "C"

// ---- measurement helper: HBM stream peak at a given read/write mix ---------
// R input arrays read and W output arrays written once per element, 16-byte
// vectors, grid-stride, one wave of resident CTAs: the bandwidth a nest with
// the same read:write mix could reach (the copy peak is R = W = 1).
struct StreamPtrs {
    const double2* in[9];
    double2* out[6];
    double* sink;   // reads-only probes: a never-taken store keeps the loads alive
};
// each CTA streams one contiguous 4 x 256 x 16-byte chunk, loads of all R
// arrays issued before any use
template <int R, int W>
__global__ void __launch_bounds__(256) stream_rw_kernel(StreamPtrs p, long long n2) {
    constexpr int U = 4;
    const long long chunk = (long long)U * blockDim.x;
    double2 tot = make_double2(0.0, 0.0);
    for (long long c0 = blockIdx.x * chunk; c0 < n2; c0 += (long long)gridDim.x * chunk) {
        double2 v[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const long long i = c0 + u * blockDim.x + threadIdx.x;
                v[u][r] = i < n2 ? p.in[r][i] : make_double2(0.0, 0.0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = c0 + u * blockDim.x + threadIdx.x;
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                acc.x += v[u][r].x;
                acc.y += v[u][r].y;
            }
            if (i < n2) {
#pragma unroll
                for (int w = 0; w < W; ++w) p.out[w][i] = make_double2(acc.x + w, acc.y - w);
            }
            tot.x += acc.x;
            tot.y += acc.y;
        }
    }
    if (W == 0 && tot.x + tot.y == 1.25e300) *p.sink = tot.x;
}
template <int R, int W>
static acs_status stream_launch(const StreamPtrs& p, long long n2, cudaStream_t s) {
    // one CTA per 4 x 256-element chunk (no grid-stride loop): the hardware
    // scheduler balances the tail, as the copy kernel of the measured peak does
    const long long blocks = (n2 + 4 * 256 - 1) / (4 * 256);
    stream_rw_kernel<R, W><<<(unsigned)blocks, 256, 0, s>>>(p, n2);
    return ACS_OK;
}
template <int R, int W>
static acs_status stream_dispatch_w(int w, const StreamPtrs& p, long long n2, cudaStream_t s) {
    if constexpr (W > 6) {
        return ACS_E_ARG;
    } else {
        if (w == W) return stream_launch<R, W>(p, n2, s);
        return stream_dispatch_w<R, W + 1>(w, p, n2, s);
    }
}
template <int R>
static acs_status stream_dispatch(int r, int w, const StreamPtrs& p, long long n2, cudaStream_t s) {
    if constexpr (R > 9) {
        return ACS_E_ARG;
    } else {
        if (r == R) return stream_dispatch_w<R, 0>(w, p, n2, s);
        return stream_dispatch<R + 1>(r, w, p, n2, s);
    }
}

extern "C" {

acs_status acs_stream_probe(int reads, int writes, int64_t elems, int reps, float* gbs_out) {
    if (reads < 1 || reads > 9 || writes < 0 || writes > 6 || elems < 2 || reps < 1 || !gbs_out) {
        set_error("acs_stream_probe: reads 1..9, writes 0..6, elems >= 2, reps >= 1");
        return ACS_E_ARG;
    }
    const long long n2 = elems / 2;
    const size_t bytes = (size_t)n2 * sizeof(double2);
    StreamPtrs p{};
    std::vector<void*> bufs;
    double* sink = nullptr;
    cudaMalloc(&sink, sizeof(double));
    p.sink = sink;
    auto cleanup = [&] {
        for (void* b : bufs) cudaFree(b);
        cudaFree(sink);
    };
    for (int i = 0; i < reads + writes; ++i) {
        void* b = nullptr;
        if (cudaMalloc(&b, bytes) != cudaSuccess) {
            cleanup();
            set_error("acs_stream_probe: cudaMalloc failed");
            return ACS_E_CUDA;
        }
        cudaMemset(b, 0, bytes);
        bufs.push_back(b);
        if (i < reads) p.in[i] = static_cast<const double2*>(b);
        else p.out[i - reads] = static_cast<double2*>(b);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> t((size_t)reps);
    acs_status st = stream_dispatch<1>(reads, writes, p, n2, nullptr);   // warm-up
    for (int i = 0; i < reps && st == ACS_OK; ++i) {
        cudaEventRecord(e0, nullptr);
        st = stream_dispatch<1>(reads, writes, p, n2, nullptr);
        cudaEventRecord(e1, nullptr);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t[i], e0, e1);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cleanup();
    if (st != ACS_OK) return st;
    std::sort(t.begin(), t.end());
    *gbs_out = (float)((double)bytes * (reads + writes) / (t[0] * 1e-3) / 1e9);   // best of reps, like the copy peak
    // (1R:1W measures 6734 GB/s on the B200 pool, vs 6557 for MEASURED_PEAKS' torch copy)
    return check_launch("acs_stream_probe");
}

acs_status acs_fill(const acs_array* a, acs_fill_kind kind, uint64_t seed, double lo, double hi, double p,
                    int64_t flat_offset, void* cuda_stream) {
    StridedDesc d;
    long long n;
    if (!make_desc(a, d, n)) {
        set_error("acs_fill: bad array descriptor");
        return ACS_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const int g = grid_for(n);
    switch (a->dtype) {
        case ACS_F64: fill_kernel<double><<<g, 256, 0, s>>>((double*)a->data, d, n, kind, seed, lo, hi, p, (long long)flat_offset); break;
        case ACS_F32: fill_kernel<float><<<g, 256, 0, s>>>((float*)a->data, d, n, kind, seed, lo, hi, p, (long long)flat_offset); break;
        case ACS_I32: fill_kernel<int><<<g, 256, 0, s>>>((int*)a->data, d, n, kind, seed, lo, hi, p, (long long)flat_offset); break;
        case ACS_U8: fill_kernel<uint8_t><<<g, 256, 0, s>>>((uint8_t*)a->data, d, n, kind, seed, lo, hi, p, (long long)flat_offset); break;
        default: set_error("acs_fill: unsupported dtype"); return ACS_E_ARG;
    }
    return check_launch("acs_fill");
}

acs_status acs_copy(const acs_array* dst, const acs_array* src, void* cuda_stream) {
    StridedDesc dd, sd;
    long long nd, ns;
    if (!make_desc(dst, dd, nd) || !make_desc(src, sd, ns) || dst->ndim != src->ndim) {
        set_error("acs_copy: bad array descriptor");
        return ACS_E_ARG;
    }
    for (int p = 0; p < dst->ndim; ++p)
        if (dst->dims[p] != src->dims[p]) {
            set_error("acs_copy: dims differ");
            return ACS_E_SHAPE;
        }
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const int g = grid_for(nd);
    const acs_dtype a = dst->dtype, b = src->dtype;
    if (a == ACS_F64 && b == ACS_F64) copy_kernel<double, double><<<g, 256, 0, s>>>((double*)dst->data, dd, (const double*)src->data, sd, nd);
    else if (a == ACS_F32 && b == ACS_F32) copy_kernel<float, float><<<g, 256, 0, s>>>((float*)dst->data, dd, (const float*)src->data, sd, nd);
    else if (a == ACS_I32 && b == ACS_I32) copy_kernel<int, int><<<g, 256, 0, s>>>((int*)dst->data, dd, (const int*)src->data, sd, nd);
    else if (a == ACS_U8 && b == ACS_I32) copy_kernel<uint8_t, int><<<g, 256, 0, s>>>((uint8_t*)dst->data, dd, (const int*)src->data, sd, nd);
    else if (a == ACS_I32 && b == ACS_U8) copy_kernel<int, uint8_t><<<g, 256, 0, s>>>((int*)dst->data, dd, (const uint8_t*)src->data, sd, nd);
    else {
        set_error("acs_copy: unsupported dtype pair");
        return ACS_E_ARG;
    }
    return check_launch("acs_copy");
}

acs_status acs_native_strides(const acs_kernel* k, const char* array_name, int ndim, const int64_t* dims,
                              int64_t* strides_out) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || !array_name || !dims || !strides_out || ndim < 1 || ndim > 8) {
        set_error("acs_native_strides: bad argument");
        return ACS_E_ARG;
    }
    // Row pitch of the innermost spatial subscript padded to 16 elements, so
    // every row starts 64/128-byte aligned and the TMA can describe the array
    // (global strides must be multiples of 16 bytes).
    auto pad = [](int64_t n) { return (n + 15) / 16 * 16; };
    bool comp = false;
    for (size_t i = 0; i < e->arrays.size(); ++i)
        if (e->arrays[i] == array_name) comp = e->component_last[i] != 0;
    const bool soa = e->soa_last_dim && ndim >= 2 && comp;
    const int inner = soa ? ndim - 2 : ndim - 1;
    int64_t st = 1;
    for (int p = inner; p >= 0; --p) {
        strides_out[p] = st;
        st *= (p == inner && ndim > 1) ? pad(dims[p]) : dims[p];
    }
    if (soa) strides_out[ndim - 1] = st;   // q-major SoA: the distribution subscript is slowest
    return ACS_OK;
}

acs_status acs_native_offset(const acs_kernel* k, const char* array_name, int elem_size, int64_t* offset_out) {
    const Entry* e = reinterpret_cast<const Entry*>(k);
    if (!e || !array_name || !offset_out || elem_size <= 0) {
        set_error("acs_native_offset: bad argument");
        return ACS_E_ARG;
    }
    *offset_out = 0;
    // Shift the array by a few elements so the first interior point of every
    // row (x = the loop's constant lower bound) starts a 32-byte sector:
    // interior rows then read and write whole sectors (no over-fetch of the
    // ghost column, no read-modify-write of a sector shared with it).  Only
    // for the D3Q19 SoA planes and entries flagged row_offset (zsolve), whose
    // fast skeletons do not use the TMA (which needs 16-byte-aligned bases).
    bool comp = false;
    for (size_t i = 0; i < e->arrays.size(); ++i)
        if (e->arrays[i] == array_name) comp = e->component_last[i] != 0;
    if (((e->soa_last_dim && comp) || e->row_offset) && e->inner_lo > 0 && 32 % elem_size == 0) {
        const int per = 32 / elem_size;
        *offset_out = (per - e->inner_lo % per) % per;
    }
    return ACS_OK;
}

}  // extern "C"
