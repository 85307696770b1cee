# zsolve: parity + tuned bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "zsolve or z_solve" 2>&1 | tail -2
timeout 900 python - <<'PY'
import json, bench
slot, name, tms = bench.tune_kernel("zsolve.c:z_solve_lhs:0", 256, "f64", "accsat")
ms, gbs, w = bench.bench_kernel("zsolve.c:z_solve_lhs:0", 256, "f64", 1, "accsat", "default", reps=5)
print(json.dumps({"slot": slot, "name": name, "tms": tms, "gbs": gbs, "frac": gbs / 6543.1}))
PY
