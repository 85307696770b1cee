mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "advec or clover" > gpurun_out/pytest_adv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_adv.log
tail -2 gpurun_out/pytest_adv.log
timeout 900 python - > gpurun_out/adv_bench.json 2> gpurun_out/adv_bench.err <<'PY'
import json, bench
kid = "clover.c:advec_cell_x:2"
slot, name, tms = bench.tune_kernel(kid, 7680, "f64", "accsat")
ms, gbs, w = bench.bench_kernel(kid, 7680, "f64", 1, "accsat", "default", reps=5)
print(json.dumps({"slot": slot, "name": name, "tms": tms, "gbs": gbs, "frac": gbs / 6543.1}))
PY
cat gpurun_out/adv_bench.json; tail -2 gpurun_out/adv_bench.err
