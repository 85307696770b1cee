/* Host-side seeded inputs for the CPU checkers — TEST INFRASTRUCTURE ONLY.
 *
 * The same counter-based SplitMix64 stream as paper_2306_13002_b200/nests.py
 * (`splitmix64`, `uniform`, `make_inputs`): element i of an array whose
 * parameter sits at position p is drawn from seed 20261017 + p, counter
 * offset + i, mapped to lo + (hi - lo) * u with u = (x >> 11) * 2^-53 (two
 * roundings; this file is compiled with -ffp-contract=off).  numpy builds
 * these arrays with ~5 full-size temporaries, which does not fit a 1024^3
 * workload; this fills in place with OpenMP, bit-identical
 * (tests/test_oracle.py::test_host_fill_matches_make_inputs).
 *
 * Used by bench.py's reference arm (--impl reference) so that arm loads
 * nothing but oracle/_ref/libacs_cpu.so.
 */
#include <stdint.h>

static inline uint64_t sm64(uint64_t seed, uint64_t idx) {
    uint64_t z = seed + (idx + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline double unit(uint64_t seed, uint64_t idx) {
    return (double)(sm64(seed, idx) >> 11) * (1.0 / 9007199254740992.0);
}

/* kind: 0 uniform [lo, hi), 1 const lo, 2 mask (u < p) as int32, 3 D3Q19
 * weights w[i % 19] * (1 + U[lo, hi)).  dtype: 0 f64, 1 f32, 2 i32. */
int acs_cpu_fill(void* dst, int64_t n, int dtype, int kind, uint64_t seed, double lo, double hi, double p,
                 int64_t offset, int threads) {
    static const double w19[19] = {1.0 / 3, 1.0 / 18, 1.0 / 18, 1.0 / 18, 1.0 / 18, 1.0 / 18, 1.0 / 18,
                                   1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36,
                                   1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36};
    if (!dst || n < 0 || dtype < 0 || dtype > 2 || kind < 0 || kind > 3) return 1;
    const double span = hi - lo;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t c = (uint64_t)(offset + i);
        double v;
        switch (kind) {
            case 0: v = lo + span * unit(seed, c); break;
            case 1: v = lo; break;
            case 2: v = unit(seed, c) < p ? 1.0 : 0.0; break;
            default: {
                const double one = 1.0 + (lo + span * unit(seed, c));
                v = w19[c % 19] * one;
            }
        }
        if (dtype == 0) ((double*)dst)[i] = v;
        else if (dtype == 1) ((float*)dst)[i] = (float)v;
        else ((int32_t*)dst)[i] = (int32_t)v;
    }
    return 0;
}
