// accsat_b200.hpp — C++ host API over the C ABI (include/accsat_b200.h).
//
// Mirrors the reference's executor interface so a satcc user switches by
// changing one call:
//
//   reference  satcc::Environment satcc::eval_region(const Stmt& body, Environment env)
//              (proj/include/satcc/interp.hpp:72-74) — tree-walks ONE body
//   here       acs::Environment  acs::eval_region(const std::string& kernel_id,
//                                                 Environment env, Variant v)
//              — runs the WHOLE registered nest on the B200
//
// The value types keep the reference's names and meaning: Scalar (tagged
// int64 / double, interp.hpp:13-24), ArrayBuf (typed row-major buffer with
// dims, interp.hpp:27-48), Environment (name-ordered maps, interp.hpp:51-54),
// VariantConfig (pipeline.hpp:14-20).  Errors throw EvalError / InternalError
// like proj/include/satcc/diag.hpp:43-53.  diff_envs applies the reference
// comparator's rule (proj/src/oracle.cpp:30-38).
//
// Header-only; link with libaccsat_b200.so and libcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "accsat_b200.h"

namespace acs {

enum class Ty { Int, Double };

struct Scalar {
    Ty type = Ty::Double;
    long long i = 0;
    double d = 0.0;
    static Scalar of_int(long long v) { return {Ty::Int, v, 0.0}; }
    static Scalar of_double(double v) { return {Ty::Double, 0, v}; }
    double as_double() const { return type == Ty::Int ? static_cast<double>(i) : d; }
};

// Like satcc::ArrayBuf, but int arrays hold the compiled nest's C `int`
// (int32) and real arrays may be fp32 (the wave4 fp32 configuration).
struct ArrayBuf {
    acs_dtype dtype = ACS_F64;
    std::vector<long long> dims;
    std::vector<double> dv;   // ACS_F64
    std::vector<float> fv;    // ACS_F32
    std::vector<int32_t> iv;  // ACS_I32
    size_t size() const {
        size_t n = 1;
        for (long long d : dims) n *= static_cast<size_t>(d);
        return n;
    }
    size_t bytes() const { return size() * (dtype == ACS_F64 ? 8 : 4); }
    void* data() { return dtype == ACS_F64 ? (void*)dv.data() : dtype == ACS_F32 ? (void*)fv.data() : (void*)iv.data(); }
    const void* data() const {
        return dtype == ACS_F64 ? (const void*)dv.data() : dtype == ACS_F32 ? (const void*)fv.data() : (const void*)iv.data();
    }
    double get(size_t at) const { return dtype == ACS_F64 ? dv[at] : dtype == ACS_F32 ? fv[at] : iv[at]; }
};

struct Environment {
    std::map<std::string, Scalar> scalars;
    std::map<std::string, ArrayBuf> arrays;
};

class EvalError : public std::runtime_error {
  public:
    explicit EvalError(const std::string& m) : std::runtime_error(m) {}
};
class InternalError : public std::logic_error {
  public:
    explicit InternalError(const std::string& m) : std::logic_error(m) {}
};

// VariantConfig names (cse, cse+sat, cse+bulk, accsat) plus the original text.
enum class Variant {
    Original = ACS_ORIGINAL,
    Cse = ACS_CSE,
    CseBulk = ACS_CSE_BULK,
    CseSat = ACS_CSE_SAT,
    AccSat = ACS_ACCSAT,
    OriginalNvcc = ACS_ORIGINAL_NVCC   // measurement baseline, not a reference form
};

inline Variant variant_from_name(const std::string& s) {
    if (s == "original") return Variant::Original;
    if (s == "cse") return Variant::Cse;
    if (s == "cse+bulk") return Variant::CseBulk;
    if (s == "cse+sat") return Variant::CseSat;
    if (s == "accsat") return Variant::AccSat;
    if (s == "original-nvcc") return Variant::OriginalNvcc;
    throw std::invalid_argument("unknown variant: " + s + " (expected original, cse, cse+sat, cse+bulk, or accsat)");
}

inline void check(acs_status s, const char* what) {
    if (s == ACS_OK) return;
    std::string m = std::string(what) + ": " + acs_last_error();
    if (s == ACS_E_CUDA || s == ACS_E_NCCL) throw InternalError(m);
    throw EvalError(m);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw InternalError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Runs the whole nest of `kernel_id` ("<file>:<function>:<region>") on the
// current CUDA device over a copy of `env` and returns the post-state.
inline Environment eval_region(const std::string& kernel_id, Environment env, Variant v = Variant::AccSat,
                               acs_schedule sched = ACS_SCHED_DEFAULT, cudaStream_t stream = nullptr) {
    const acs_kernel* k = nullptr;
    check(acs_lookup(kernel_id.c_str(), &k), "acs_lookup");
    acs_kernel_info info{};
    check(acs_kernel_get_info(k, &info), "acs_kernel_get_info");
    std::vector<acs_array> arrs(info.n_arrays);
    std::vector<void*> dev(info.n_arrays, nullptr);
    std::vector<std::string> names(info.n_arrays);
    struct Guard {
        std::vector<void*>& p;
        ~Guard() {
            for (void* x : p)
                if (x) cudaFree(x);
        }
    } guard{dev};
    for (int a = 0; a < info.n_arrays; ++a) {
        names[a] = acs_kernel_array_name(k, a);
        auto it = env.arrays.find(names[a]);
        if (it == env.arrays.end()) throw EvalError("read of undefined array: " + names[a]);
        ArrayBuf& b = it->second;
        cuda_check(cudaMalloc(&dev[a], b.bytes()), "cudaMalloc");
        cuda_check(cudaMemcpyAsync(dev[a], b.data(), b.bytes(), cudaMemcpyHostToDevice, stream), "H2D");
        acs_array& d = arrs[a];
        d = acs_array{};
        d.name = names[a].c_str();
        d.dtype = b.dtype;
        d.ndim = static_cast<int32_t>(b.dims.size());
        for (size_t p = 0; p < b.dims.size(); ++p) d.dims[p] = b.dims[p];
        d.data = dev[a];
    }
    std::vector<acs_scalar> sc(info.n_scalars);
    std::vector<std::string> snames(info.n_scalars);
    for (int s = 0; s < info.n_scalars; ++s) {
        snames[s] = acs_kernel_scalar_name(k, s);
        auto it = env.scalars.find(snames[s]);
        if (it == env.scalars.end()) throw EvalError("read of undefined variable: " + snames[s]);
        sc[s].name = snames[s].c_str();
        sc[s].is_int = it->second.type == Ty::Int;
        sc[s].i = it->second.i;
        sc[s].d = it->second.d;
    }
    check(acs_launch(k, static_cast<acs_variant>(v), sched, arrs.data(), info.n_arrays, sc.data(), info.n_scalars, stream),
          "acs_launch");
    for (int a = 0; a < info.n_arrays; ++a) {
        ArrayBuf& b = env.arrays[names[a]];
        cuda_check(cudaMemcpyAsync(b.data(), dev[a], b.bytes(), cudaMemcpyDeviceToHost, stream), "D2H");
    }
    cuda_check(cudaStreamSynchronize(stream), "sync");
    return env;
}

// The reference comparator (proj/src/oracle.cpp:30-38): a value passes when
// |got-want| <= tol_rel*max(|got|,|want|) or <= 1e-12; NaN never passes.
struct DiffReport {
    double max_rel_err = 0.0, max_abs_err = 0.0;
    long long failures = 0;
    bool ok() const { return failures == 0; }
};

// nan_equal: NaN matches NaN (any payload) and an infinity matches the same
// infinity — for edge-value inputs, where the reference rule (NaN always
// fails) cannot tell a faithful executor from a broken one.
inline DiffReport diff_envs(const Environment& want, const Environment& got, double tol_rel, double abs_floor = 1e-12,
                            bool nan_equal = false) {
    DiffReport rep;
    auto value = [&](double w, double g) {
        if (nan_equal && ((std::isnan(w) && std::isnan(g)) || (std::isinf(w) && w == g))) return;
        const double ae = std::fabs(g - w), mag = std::max(std::fabs(g), std::fabs(w));
        const double re = mag > 0.0 ? ae / mag : 0.0;
        rep.max_abs_err = std::max(rep.max_abs_err, ae);
        rep.max_rel_err = std::max(rep.max_rel_err, re);
        if (!(ae <= tol_rel * mag || ae <= abs_floor)) rep.failures++;
    };
    for (auto& [n, v] : want.scalars) {
        auto it = got.scalars.find(n);
        if (it == got.scalars.end()) rep.failures++;
        else value(v.as_double(), it->second.as_double());
    }
    for (auto& [n, v] : want.arrays) {
        auto it = got.arrays.find(n);
        if (it == got.arrays.end() || it->second.dims != v.dims) {
            rep.failures++;
            continue;
        }
        for (size_t i = 0; i < v.size(); ++i) value(v.get(i), it->second.get(i));
    }
    return rep;
}

}  // namespace acs
