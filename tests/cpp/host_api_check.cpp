// C++ host API check (include/accsat_b200.hpp): the call a satcc maintainer
// would make in place of satcc::eval_region (proj/src/interp.cpp:266-270).
// Builds a small jacobi7 Environment, runs the whole nest on the GPU in the
// original and accsat forms, and checks the post-state bit for bit against a
// plain C++ restatement of the nest text (two roundings per operation, the
// text's evaluation order; compiled with -ffp-contract=off), plus the
// reference comparator rule and the EvalError contract.
// Usage: host_api_check  -> prints "host_api_check ok" and exits 0.
#include <cstdio>
#include <cstring>
#include <string>

#include "accsat_b200.hpp"

static double u01(unsigned long long& s) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return (double)(s >> 11) * (1.0 / 9007199254740992.0);
}

int main() {
    const int nz = 9, ny = 11, nx = 37;
    const long long Z = nz + 2, Y = ny + 2, X = nx + 2;
    acs::Environment env;
    acs::ArrayBuf a0;
    a0.dtype = ACS_F64;
    a0.dims = {Z, Y, X};
    a0.dv.resize(a0.size());
    unsigned long long seed = 20261017ULL;
    for (double& v : a0.dv) v = u01(seed);
    acs::ArrayBuf an = a0;
    env.arrays["A0"] = a0;
    env.arrays["Anext"] = an;
    const double c0 = 1.0 / 6.0, c1 = 1.0 / 36.0;
    env.scalars["c0"] = acs::Scalar::of_double(c0);
    env.scalars["c1"] = acs::Scalar::of_double(c1);
    env.scalars["kbeg"] = acs::Scalar::of_int(1);
    env.scalars["kend"] = acs::Scalar::of_int(nz + 1);
    env.scalars["ny"] = acs::Scalar::of_int(Y);
    env.scalars["nx"] = acs::Scalar::of_int(X);

    // expected: nests/jacobi7.c restated
    acs::Environment want = env;
    auto at = [&](long long k, long long j, long long i) { return (k * Y + j) * X + i; };
    const std::vector<double>& A = env.arrays["A0"].dv;
    std::vector<double>& W = want.arrays["Anext"].dv;
    for (long long k = 1; k < nz + 1; ++k)
        for (long long j = 1; j < Y - 1; ++j)
            for (long long i = 1; i < X - 1; ++i) {
                double s = A[at(k + 1, j, i)] + A[at(k - 1, j, i)];
                s = s + A[at(k, j + 1, i)];
                s = s + A[at(k, j - 1, i)];
                s = s + A[at(k, j, i + 1)];
                s = s + A[at(k, j, i - 1)];
                const double t = s * c1;
                const double u = A[at(k, j, i)] * c0;
                W[at(k, j, i)] = t - u;
            }

    int fails = 0;
    for (acs::Variant v : {acs::Variant::Original, acs::Variant::AccSat}) {
        acs::Environment got = acs::eval_region("jacobi7.c:jacobi7:0", env, v);
        const std::vector<double>& G = got.arrays["Anext"].dv;
        if (std::memcmp(G.data(), W.data(), W.size() * sizeof(double)) != 0) {
            std::printf("variant %d: Anext differs bitwise\n", (int)v);
            ++fails;
        }
        acs::DiffReport rep = acs::diff_envs(want, got, 1e-12);
        if (!rep.ok()) {
            std::printf("variant %d: comparator failures %lld\n", (int)v, rep.failures);
            ++fails;
        }
    }
    // comparator modes: NaN always fails the reference rule; nan_equal accepts
    // NaN vs NaN and equal infinities, and still rejects NaN vs a number
    {
        acs::Environment a, b, c;
        a.scalars["x"] = acs::Scalar::of_double(std::nan(""));
        b.scalars["x"] = acs::Scalar::of_double(-std::nan(""));
        c.scalars["x"] = acs::Scalar::of_double(1.0);
        a.scalars["y"] = b.scalars["y"] = c.scalars["y"] = acs::Scalar::of_double(HUGE_VAL);
        if (acs::diff_envs(a, b, 1e-12).ok() || !acs::diff_envs(a, b, 1e-12, 1e-12, true).ok() ||
            acs::diff_envs(a, c, 1e-12, 1e-12, true).ok()) {
            std::printf("diff_envs nan_equal mode wrong\n");
            ++fails;
        }
    }
    // EvalError contract: a missing array is an error, never a silent result
    acs::Environment bad = env;
    bad.arrays.erase("Anext");
    bool threw = false;
    try {
        acs::eval_region("jacobi7.c:jacobi7:0", bad, acs::Variant::AccSat);
    } catch (const acs::EvalError&) {
        threw = true;
    }
    if (!threw) {
        std::printf("missing array did not raise EvalError\n");
        ++fails;
    }
    if (fails) return 1;
    std::printf("host_api_check ok\n");
    return 0;
}
