# parity (pytest -k $1) + tuned bench of one nest: bash tools/gpu/nest_check.sh <pytest -k expr> <kernel_id> <size> <dtype> <sweeps>
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$1" 2>&1 | tail -1
timeout 900 python - "$2" "$3" "$4" "$5" <<'PY'
import json, sys, bench
kid, size, dt, sw = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
slot, name, tms = bench.tune_kernel(kid, size, dt, "accsat")
ms, gbs, w = bench.bench_kernel(kid, size, dt, sw, "accsat", "default", reps=5)
print(json.dumps({"slot": slot, "name": name, "tms": {k: round(v, 4) for k, v in tms.items()}, "gbs": round(gbs, 1), "frac": round(gbs / 6543.1, 4)}))
PY
