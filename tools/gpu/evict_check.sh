# L2 evict_first on the once-read TMA streams (ACS_TMA_EVICT=1) vs default: parity of the march
# slots, then interleaved bench lines (headline + per-kernel table) in alternating processes.
mkdir -p gpurun_out
ACS_TMA_EVICT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/evict_pytest.log 2>&1
rc=$?; echo "parity (evict) rc=$rc $(tail -1 gpurun_out/evict_pytest.log)"; [ $rc -eq 0 ] || exit 1
for rep in 1 2 3; do for ev in 0 1; do
  ACS_TMA_EVICT=$ev timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/evict_$ev_$rep.json 2>/dev/null
  python - <<PY
import json
d=json.loads(open("gpurun_out/evict_$ev_$rep.json").read().strip().splitlines()[-1])
pk=d["per_kernel"]
print("evict $ev rep $rep headline", d["value"], "|", " ".join(f"{k}:{v['accsat/tuned']['gbs']:.0f}" for k,v in pk.items() if isinstance(v,dict) and 'accsat/tuned' in v))
PY
done; done | tee gpurun_out/evict_check.txt
