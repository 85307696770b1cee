timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "jacobi or wave4 or calc or shard" 2>&1 | tail -2
for pdl in 1 0; do
ACS_PDL=$pdl timeout 900 python - <<'PY'
import json, os, bench
out = {}
bench.tune_kernel("jacobi7.c:jacobi7:0", 256, "f64", "accsat")
ms, gbs, w = bench.bench_kernel("jacobi7.c:jacobi7:0", 256, "f64", 100, "accsat", "default", reps=5)
print("PDL", os.environ.get("ACS_PDL"), round(ms, 4), round(gbs, 1), round(gbs / 6543.1, 4))
PY
done
