mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "jacobi or wave4" > gpurun_out/pytest_rb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rb.log
tail -3 gpurun_out/pytest_rb.log
timeout 900 python - > gpurun_out/rb_bench.json 2> gpurun_out/rb_bench.err <<'PY'
import json, bench
peak = 6543.1
out = {}
for kid, size, dt, sw in (("jacobi7.c:jacobi7:0", 256, "f64", 100), ("wave4.c:wave4:0", 1024, "f32", 1)):
    slot, name, tms = bench.tune_kernel(kid, size, dt, "accsat")
    ms, gbs, w = bench.bench_kernel(kid, size, dt, sw, "accsat", "default", reps=5)
    out[kid] = {"slot": slot, "name": name, "tms": tms, "gbs": gbs, "frac": gbs / peak}
print(json.dumps(out))
PY
cat gpurun_out/rb_bench.json; tail -3 gpurun_out/rb_bench.err
