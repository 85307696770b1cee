/*
 * accsat_b200.h — C ABI of the B200 loop-nest execution backend.
 *
 * Drop-in boundary for the reference's execution path (arXiv 2306.13002,
 * ACC Saturator / satcc).  The reference runs a nest either in process with
 * its interpreter
 *     Environment eval_region(const Stmt& body, Environment env)
 *         (proj/include/satcc/interp.hpp:72-74, proj/src/interp.cpp:266-270)
 * or out of process by handing the emitted C to a compiler
 *     satcc [flags] -- cc -O3 kernel.c   (proj/tools/satcc_main.cpp:285-360).
 * This library replaces both with hand-written sm_100a kernels.  Plain C
 * types only: no C++ types or exceptions cross it.
 *
 *   - A kernel is registered under "<file>:<function>:<region index>", the key
 *     find_regions assigns (proj/src/ast.cpp:390-398, Region::index).
 *   - A variant is a VariantConfig name (proj/include/satcc/pipeline.hpp:14-20)
 *     plus ORIGINAL (the unoptimized source text).
 *   - Arrays are caller-owned DEVICE buffers described like ArrayBuf
 *     (proj/include/satcc/interp.hpp:27-48): element type, dims, and element
 *     strides (0 = row-major, i.e. ArrayBuf::flat).  Scalars are named
 *     int64/double values like Scalar (interp.hpp:13-24).
 *   - Errors: a status code plus a thread-local message (acs_last_error), the
 *     analogue of EvalError / InternalError (proj/include/satcc/diag.hpp:43-53).
 *     There is no CPU fallback: a kernel that is not registered, or a CUDA
 *     failure, is an error.
 *   - Launches are asynchronous on the caller's stream; registry lookups are
 *     thread-safe.
 */
#ifndef ACCSAT_B200_H
#define ACCSAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACS_ABI_VERSION 1
#define ACS_MAX_DIMS 8

typedef enum {
    ACS_OK = 0,
    ACS_E_ARG = 1,        /* bad argument: null pointer, unknown name, missing array/scalar */
    ACS_E_NO_KERNEL = 2,  /* kernel id / variant / schedule not registered */
    ACS_E_SHAPE = 3,      /* dims, strides or dtype do not match the kernel's declaration */
    ACS_E_CUDA = 4,       /* CUDA runtime error (message has the CUDA error string) */
    ACS_E_NCCL = 5,       /* peer / collective setup error */
    ACS_E_BOUNDS = 6,     /* iteration space would index outside an array (EvalError analogue) */
    ACS_E_LAYOUT = 7      /* an explicitly requested schedule slot cannot describe these arrays'
                             layout (e.g. the TMA needs 16-byte aligned bases and pitches); the
                             DEFAULT schedule never fails this way (it runs the naive skeleton) */
} acs_status;

typedef enum { ACS_F64 = 0, ACS_F32 = 1, ACS_I32 = 2, ACS_I64 = 3, ACS_U8 = 4 } acs_dtype;

/* Forms of a nest: the original source, and the four VariantConfig outputs of
 * the reference optimizer (pipeline.cpp:97-110). */
typedef enum {
    ACS_ORIGINAL = 0,
    ACS_CSE = 1,
    ACS_CSE_BULK = 2,
    ACS_CSE_SAT = 3,
    ACS_ACCSAT = 4,
    /* Measurement baseline, not a reference form: the ORIGINAL text compiled
     * the way nvcc does by default (plain C arithmetic with FMA contraction
     * left to the compiler, loads free to be cached / CSE'd) — how much of the
     * saturation win a production compiler recovers on its own (SURVEY.md §7
     * hard part 1).  Naive schedule only; results agree with the reference
     * within the comparator tolerance, not bit for bit. */
    ACS_ORIGINAL_NVCC = 5
} acs_variant;

/* Kernel skeleton: NAIVE = one thread per point, every array reference of the
 * form is its own global load in source order (what a directive compiler
 * makes of the text); TILED = the B200 marching-tile skeleton (TMA boxes of
 * every loaded array staged in a shared-memory ring ahead of compute).
 * DEFAULT = NAIVE for ORIGINAL (faithful baseline) and the preferred slot
 * (first tiled configuration, or the acs_tune winner) otherwise. */
typedef enum { ACS_SCHED_DEFAULT = 0, ACS_SCHED_NAIVE = 1, ACS_SCHED_TILED = 2 } acs_schedule;
/* ACS_SCHED_SLOT(i): an explicit registered configuration (slot 0 = naive,
 * slots 1.. = tiled configurations, see acs_kernel_schedule_name). */
#define ACS_SCHED_SLOT(i) ((acs_schedule)(16 + (i)))

typedef struct {
    const char* name;              /* parameter name in the nest text */
    acs_dtype dtype;
    int32_t ndim;
    int64_t dims[ACS_MAX_DIMS];
    int64_t strides[ACS_MAX_DIMS]; /* in elements; all zero = row-major (reference layout) */
    void* data;                    /* device pointer */
} acs_array;

typedef struct {
    const char* name;
    int32_t is_int;                /* 1: use i, 0: use d */
    int64_t i;
    double d;
} acs_scalar;

typedef struct acs_kernel acs_kernel;  /* opaque registry entry */

typedef struct {
    const char* kernel_id;         /* "<file>:<function>:<region>" */
    const char* function;
    int32_t region;
    int32_t n_loops;               /* marked loops = GPU iteration space */
    int32_t n_arrays;
    int32_t n_scalars;
    int32_t static_loads[5];       /* per acs_variant: array reads per point (count_static_loads) */
    int32_t fma_count[5];          /* per acs_variant: single-rounding FMAs per point */
    int32_t has_tiled;             /* a TILED skeleton is registered */
    int32_t has_f32;               /* an fp32 instantiation is registered */
    int32_t n_schedules;           /* registered slots (naive + tiled configurations), fp64 */
} acs_kernel_info;

int acs_abi_version(void);
const char* acs_last_error(void);

/* Registry (kernel registration by find_regions key). */
int acs_kernel_count(void);
const char* acs_kernel_id(int index);
acs_status acs_lookup(const char* kernel_id, const acs_kernel** out);
acs_status acs_kernel_get_info(const acs_kernel* k, acs_kernel_info* out);
const char* acs_kernel_array_name(const acs_kernel* k, int index);
const char* acs_kernel_scalar_name(const acs_kernel* k, int index);
int acs_kernel_scalar_is_int(const acs_kernel* k, int index);

/* Subscript-0 reach of one array (kernel parameter order `index`): the
 * min/max static offset, relative to the outermost loop variable, of its
 * loads (*ld_lo, *ld_hi) and of its stores (*st_lo, *st_hi); *sliced = 1 when
 * subscript 0 follows the outermost loop (the array can be cut into slabs).
 * Flags *loaded / *stored say whether the nest reads / writes it at all. */
acs_status acs_kernel_array_reach(const acs_kernel* k, int index, int* sliced, int* loaded, int* stored,
                                  int* ld_lo, int* ld_hi, int* st_lo, int* st_hi);

/* Unconditional static store targets of array `index`: the elements the nest
 * writes at EVERY point of its iteration space on every path (a store in
 * both arms of an if counts; the intersection over all five forms).  Target i
 * is offsets[i*ACS_MAX_DIMS + p]: for a subscript that follows a loop variable
 * the constant offset from it, for an absolute subscript the constant;
 * loop_of[p] (optional, ACS_MAX_DIMS entries) = that loop's index, or -1.  Lets a
 * host-buffer caller skip uploading elements the launch overwrites (the
 * eval_region contract, proj/src/interp.cpp:266-270, returns every element:
 * unwritten ones keep their input value).  *n_targets = total count; at most
 * max_targets are written. */
acs_status acs_kernel_must_write(const acs_kernel* k, int index, int32_t* loop_of, int max_targets,
                                 int32_t* offsets, int* n_targets);

/* Iteration space of the marked loops (n_loops entries, outermost first,
 * half-open [lo, hi)) that acs_launch would run for these scalars — the
 * parsed init/for_cond of each For (proj/include/satcc/ast.hpp:114-118). */
acs_status acs_kernel_iteration_space(const acs_kernel* k, const acs_scalar* scalars, int n_scalars, int64_t* lo,
                                      int64_t* hi);

/* Copies the box [box_lo, box_hi) of a row-major array (identical dims on both
 * sides) between host and device memory: kind 0 = host->device, 1 =
 * device->host, 2 = device->device, 3 = inferred (unified addressing).
 * Asynchronous on `cuda_stream` (pinned host memory for overlap); trailing
 * full positions are fused into one contiguous run, three positions per
 * DMA descriptor (cudaMemcpy3DAsync). */
acs_status acs_copy_box(void* dst, const void* src, int elem_size, int ndim, const int64_t* dims,
                        const int64_t* box_lo, const int64_t* box_hi, int kind, void* cuda_stream);

/* Runs the WHOLE nest (every marked loop) of one region on `stream`.
 * Arrays/scalars are matched to the nest's parameters by name. */
acs_status acs_launch(const acs_kernel* k, acs_variant variant, acs_schedule schedule,
                      const acs_array* arrays, int n_arrays,
                      const acs_scalar* scalars, int n_scalars, void* cuda_stream);

/* Name of schedule slot `slot` for precision 0 (fp64) / 1 (fp32); NULL if absent. */
const char* acs_kernel_schedule_name(const acs_kernel* k, int precision, int slot);

/* Autotuning: times every registered slot for this variant on these arrays
 * (one warm-up each, then `reps` rounds launching every slot once — interleaved, so clock drift
 * hits all slots alike — and the median launch time per slot; the arrays are updated as by
 * repeated launches), records the fastest as what ACS_SCHED_DEFAULT /
 * ACS_SCHED_TILED use for this (kernel, precision, variant) from now on, and
 * returns it.  ms_per_launch[slot] (optional, kMaxSched=8 entries) receives
 * the timings (negative = slot absent).  Synchronous. */
acs_status acs_tune(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                    const acs_scalar* scalars, int n_scalars, void* cuda_stream, int reps, int* best_slot,
                    float* ms_per_launch);

/* ---- slab sharding across GPUs -------------------------
 * Each rank owns planes [own_lo, own_hi) (global coordinates) of the outermost
 * loop; its buffers hold those planes plus halos, local index 0 = global
 * `origin`.  Owner computes; every store of a listed array to global plane g
 * is ALSO written, from inside the same kernel, into the lower neighbour's
 * buffer when g < own_lo + halo and into the upper neighbour's when
 * g >= own_hi - halo (peer device memory: NVLink P2P, or the same device).
 * `halo` is how far beyond its owned range the NEXT step reads the produced
 * data (wave4: 2, jacobi7: 1, D3Q19 push-stream: 0 — only pushes into the
 * neighbour's planes travel; swim / CloverLeaf multi-kernel steps: 1).  No
 * store is forwarded below the upper neighbour's `hi_origin` (its first
 * buffer plane), so slabs whose stores reach past the owned range (swim's
 * j+1 stores) stay inside the neighbour's buffer.  Order steps across ranks with acs_signal /
 * acs_wait (device-side release/acquire flags, no host round trip).
 * Neighbours' buffers must have the same element strides as this rank's
 * (allocate every slab with the same plane count; use views for the rest). */
#define ACS_MAX_SHARDED 16
typedef struct {
    int64_t own_lo, own_hi;
    int64_t origin;
    int32_t halo;
    int32_t n_sharded;
    const char* names[ACS_MAX_SHARDED];   /* arrays whose stores are written through */
    void* lo_data[ACS_MAX_SHARDED];       /* lower neighbour's buffer of names[i] (NULL: none) */
    void* hi_data[ACS_MAX_SHARDED];       /* upper neighbour's buffer (NULL: none) */
    int64_t lo_origin, hi_origin;         /* neighbours' `origin` */
} acs_shard;

acs_status acs_launch_sharded(const acs_kernel* k, acs_variant variant, acs_schedule schedule,
                              const acs_array* arrays, int n_arrays, const acs_scalar* scalars, int n_scalars,
                              const acs_shard* shard, void* cuda_stream);
/* stream-ordered: after all prior work on the stream, system-scope release
 * store of `value` into each non-NULL flag (peer or local device memory) */
acs_status acs_signal(uint64_t* flag_a, uint64_t* flag_b, uint64_t value, void* cuda_stream);
/* stream-ordered: block the stream until each non-NULL local flag >= value
 * (acquire); traps after `timeout_ms` so a lost peer is a loud error, not a hang */
acs_status acs_wait(const uint64_t* flag_a, const uint64_t* flag_b, uint64_t value, int timeout_ms,
                    void* cuda_stream);
/* Graph-capturable step ordering: the step number lives in a device counter
 * (one uint64 per rank, zero before the first step).  acs_wait_ctr blocks the
 * stream until each non-NULL local flag >= *counter; acs_signal_ctr increments
 * *counter after all prior work on the stream and release-stores the new value
 * into each non-NULL (peer) flag.  A (wait_ctr, launch, signal_ctr) sequence
 * captured once in a CUDA graph is valid for every step. */
acs_status acs_signal_ctr(uint64_t* flag_a, uint64_t* flag_b, uint64_t* counter, void* cuda_stream);
acs_status acs_wait_ctr(const uint64_t* flag_a, const uint64_t* flag_b, const uint64_t* counter, int timeout_ms,
                        void* cuda_stream);
/* Time stepping of a ping-pong nest (jacobi7: A0 <-> Anext): `nsteps` steps
 * of the nest's time loop, each step reading the buffer the previous one
 * wrote (step 0 reads the array the nest reads).  blocked != 0 runs two steps
 * per launch where a temporal-blocking skeleton is registered (one pass over
 * HBM per two steps, bit-identical results); otherwise one DEFAULT launch per
 * step.  *latest = the index in `arrays` of the buffer holding the newest
 * field (with blocking the other buffer does not hold the previous step). */
acs_status acs_launch_steps(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                            const acs_scalar* scalars, int n_scalars, int nsteps, int blocked, void* cuda_stream,
                            int* latest);

/* Two time steps of a 3-level leapfrog nest (wave4: un = f(u, up, vel2), the
 * time loop rotating up <- u <- un) in ONE launch (temporal blocking,
 * kernels/tbwave.cuh).  Step 1 is written to `un` as a single step would;
 * step 2 goes to `un2`, a fourth buffer of un's dims / strides (the loop's
 * free buffer, up, is still read by neighbouring tiles' step 1).  After the
 * call the loop's state is up = un, u = un2 — the same values two
 * acs_launch calls with the rotation produce, bit for bit, provided every
 * rotating buffer (u, up, un, un2) carries the same fixed boundary (the
 * cells outside the iteration space, never written by the nest).  Replaces two
 * iterations of the nest's time loop (the reference runs one step per
 * eval_region, proj/src/interp.cpp:266-270).  ACS_E_NO_KERNEL when the nest
 * or precision has no two-step kernel; ACS_E_LAYOUT when the TMA cannot
 * describe the arrays. */
acs_status acs_launch_leapfrog2(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                                const acs_scalar* scalars, int n_scalars, const acs_array* un2, void* cuda_stream);
/* eval_region for HOST arrays (row-major, the reference layout; `data` =
 * host pointers): uploads every array, runs the whole nest with the DEFAULT
 * schedule, downloads every array the nest stores, synchronously.  The call a
 * program compiled through the B200 wrapper hand-off makes in place of the
 * nest's loops (paper_2306_13002_b200/jit.py). */
acs_status acs_eval_host(const acs_kernel* k, acs_variant variant, const acs_array* host_arrays, int n_arrays,
                         const acs_scalar* scalars, int n_scalars);
/* Loads the code of every schedule slot of (kernel, variant) for these arrays
 * without launching anything.  CUDA lazy loading loads a kernel at its first
 * launch and may wait for the device to drain: call this before a sharded
 * time loop whose acs_wait_ctr kernels spin while other streams launch. */
acs_status acs_preload(const acs_kernel* k, acs_variant variant, const acs_array* arrays, int n_arrays,
                       const acs_scalar* scalars, int n_scalars);
/* CUDA IPC of a device pointer inside any allocation (base handle + offset) */
acs_status acs_ipc_export(const void* dptr, void* handle_out /* 64 bytes */, int64_t* offset_out);
acs_status acs_ipc_import(const void* handle /* 64 bytes */, int64_t offset, void** dptr_out);
acs_status acs_ipc_close(void* dptr, int64_t offset);

/* Measurement helper (not the hot path): HBM bandwidth of a pure stream with
 * `reads` input and `writes` output arrays of `elems` doubles each (best of
 * `reps`, GB/s) — the peak a nest with the same read:write mix can reach. */
acs_status acs_stream_probe(int reads, int writes, int64_t elems, int reps, float* gbs_out);

/* Device data utilities (synthetic inputs, layout remaps). */
typedef enum { ACS_FILL_UNIFORM = 0, ACS_FILL_CONST = 1, ACS_FILL_MASK = 2, ACS_FILL_D3Q19 = 3 } acs_fill_kind;
/* Fills a (possibly strided) array.  Element at reference flat index f gets
 * SplitMix64(seed, f + flat_offset): UNIFORM lo+(hi-lo)*u, CONST lo, MASK
 * (u < p), D3Q19 w[f % 19] * (1 + (lo+(hi-lo)*u)).  Bit-identical to
 * nests.make_inputs; flat_offset lets a slab reproduce its part of a global
 * array. */
acs_status acs_fill(const acs_array* a, acs_fill_kind kind, uint64_t seed, double lo, double hi,
                    double p, int64_t flat_offset, void* cuda_stream);
/* Strided element copy between two arrays of the same dims (any strides,
 * dtype conversion between integer types or between real types). */
acs_status acs_copy(const acs_array* dst, const acs_array* src, void* cuda_stream);
/* Backend-preferred strides for an array of `kernel` (e.g. q-major SoA for the
 * D3Q19 distribution arrays); row-major otherwise. */
acs_status acs_native_strides(const acs_kernel* k, const char* array_name, int ndim,
                              const int64_t* dims, int64_t* strides_out);

/* Element offset the backend prefers for the start of array `array_name`
 * (0 for most arrays): q-major SoA component planes are shifted so the first
 * interior point of every row starts a 32-byte sector.  Allocate
 * offset + span elements and pass data + offset as acs_array.data. */
acs_status acs_native_offset(const acs_kernel* k, const char* array_name, int elem_size, int64_t* offset_out);

#ifdef __cplusplus
}
#endif
#endif /* ACCSAT_B200_H */
