mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "zsolve or z_solve" > gpurun_out/pytest_zs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zs.log
tail -3 gpurun_out/pytest_zs.log
timeout 900 python - > gpurun_out/zs_bench.json 2> gpurun_out/zs_bench.err <<'PY'
import json, bench
peak = 6543.1
row = {}
slot, name, tms = bench.tune_kernel("zsolve.c:z_solve_lhs:0", 256, "f64", "accsat")
row["tuned"] = {"slot": slot, "schedule": name, "ms": tms}
for v, s in (("original", "naive"), ("accsat", "naive"), ("accsat", "default")):
    ms, gbs, w = bench.bench_kernel("zsolve.c:z_solve_lhs:0", 256, "f64", 1, v, s, reps=5)
    row[f"{v}/{s}"] = {"ms": ms, "gbs": gbs, "frac": gbs / peak}
print(json.dumps(row))
PY
cat gpurun_out/zs_bench.json; tail -3 gpurun_out/zs_bench.err
