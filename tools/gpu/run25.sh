mkdir -p gpurun_out
timeout 900 python - > gpurun_out/jac_graph.json 2> gpurun_out/jac_graph.err <<'PY'
import json, bench
out = {}
for v, s in (("original", "naive"), ("accsat", "naive"), ("accsat", "default")):
    if s == "default":
        bench.tune_kernel("jacobi7.c:jacobi7:0", 256, "f64", "accsat")
    ms, gbs, w = bench.bench_kernel("jacobi7.c:jacobi7:0", 256, "f64", 100, v, s, reps=3)
    out[f"{v}/{s}"] = {"ms": ms, "gbs": gbs, "frac": gbs / 6543.1}
print(json.dumps(out))
PY
cat gpurun_out/jac_graph.json; tail -3 gpurun_out/jac_graph.err
