/*
 * accsat_opt.h — host stage (a): the compile-time optimizer that produces the
 * saturated form the B200 kernels execute, re-implemented in C++ for the
 * host.
 *
 * Replaces, with the same inputs, outputs and metrics:
 *   optimize_source(source, name, VariantConfig, PipelineLimits)
 *       (proj/include/satcc/pipeline.hpp:64-66, proj/src/pipeline.cpp:140-194)
 * i.e. parse -> find_regions -> per region: value-numbered SSA with per-base
 * load epochs and same-scope store->load forwarding (proj/src/ssa.cpp) ->
 * e-graph (hash-consing = load CSE, proj/src/egraph.cpp) -> [saturation with
 * the nine Table-I rules + constant folding, proj/src/rules.cpp:123-251] ->
 * extraction under the same cost model (const 0 / leaf 1 / op 10 /
 * load-div-mod-call 100, proj/src/cost.cpp:9-41) -> depth-one temps and
 * [bulk load motion] -> re-emitted module text.  Fail-open per region.
 *
 * Extraction: greedy tree-cost followed by an exact incremental DAG-cost local
 * search (milliseconds), then, when exact_time_s > 0 and a solver is
 * registered, the exact 0/1 ILP (method "ilp" when proven optimal, in place
 * of the reference's branch and bound); results are checked against the frozen
 * reference outputs for objective, load count and semantics (tests/test_opt.py).
 */
#ifndef ACCSAT_OPT_H
#define ACCSAT_OPT_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    long max_nodes;        /* saturation node budget (reference default 10000) */
    double max_time_s;     /* saturation wall-time budget (default 10) */
    int max_iters;         /* saturation iterations (default 10) */
    int dag_search;        /* 1: DAG-cost local search after greedy (default), 0: greedy only */
    double exact_time_s;   /* > 0: exact extraction through the registered solver (acs_opt_set_solver) with this
                              time limit per region; 0: off.  The reference's extract.max_time (30 s default) */
} acs_opt_limits;

/* Optimizes every directive-marked region of `source` for `variant`
 * ("cse", "cse+sat", "cse+bulk", "accsat").  On success *text_out holds the
 * emitted module and *json_out a satcc-metrics-v1 document (free both with
 * acs_opt_free).  Returns 0, or 1 with *json_out = {"error": ...} when the
 * source does not parse (per-region failures are fail-open: the region is
 * left untouched and its metrics carry the error). */
int acs_opt_optimize(const char* source, const char* name, const char* variant, const acs_opt_limits* limits,
                     char** text_out, char** json_out);
/* Differential verification of the optimized form, the reference's
 * `satcc verify` (proj/tools/satcc_main.cpp:217-283, diff_test in
 * proj/src/oracle.cpp:12-81): for every region, `trials` random environments
 * (trial t seeded t + 1; ints U[1, 8], doubles U[-10, 10], mt19937_64) run
 * the ORIGINAL and the OPTIMIZED region body under the reference's C
 * semantics (two-rounding fma, bounds-checked arrays, 50M-tick budget); every
 * scalar and array element of the original's post-state must agree within
 * tol_rel * max(|a|, |b|) or 1e-12 (NaN never passes; an error is a failure).
 * *json_out = {"file", "variant", "regions": [{region, function, n_trials,
 * max_rel_err, max_abs_err, n_failures, failures: [{seed, location, got,
 * want}] (first 10), ok}]} (free with acs_opt_free).  Returns 0 when every
 * region passes, 1 when one fails, 2 on a parse / argument error. */
int acs_opt_verify(const char* source, const char* name, const char* variant, const acs_opt_limits* limits, int trials,
                   double tol_rel, char** json_out);
void acs_opt_free(char* p);
/* Exact extraction (the reference's extract_ilp, proj/src/extract.cpp:202-241):
 * the min-DAG-cost selection over the classes reachable from the roots as a
 * 0/1 ILP.  n_nodes nodes, node i in class node_class[i] (0..n_classes-1) with
 * cost node_cost[i] and kid classes kids[kid_ptr[i] .. kid_ptr[i+1]); the root
 * classes must each select a node.  The solver writes chosen[i] (0/1) and a
 * lower bound on the optimum, and returns 0 = proven optimal, 1 = time limit
 * (chosen is feasible), 2 = no solution.  satopt.py registers HiGHS
 * (scipy.optimize.milp); with no solver registered exact_time_s is ignored. */
typedef int (*acs_opt_solver)(int n_nodes, int n_classes, const int* node_class, const long long* node_cost,
                              const int* kid_ptr, const int* kids, int n_roots, const int* roots, double time_limit_s,
                              int* chosen, double* bound);
void acs_opt_set_solver(acs_opt_solver fn);

#ifdef __cplusplus
}
#endif
#endif /* ACCSAT_OPT_H */
