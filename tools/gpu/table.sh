# GPU tests + smoke + the per-nest table (no e2e / cpu legs)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_tab.json 2> gpurun_out/bench_tab.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_tab.json'))
print("headline", d['value'], d['roofline']['frac'])
for k,r in d['per_kernel'].items():
    print(f"{k:14s} orig {r['original/naive'].get('gbs')} nvcc {r['original-nvcc/naive'].get('gbs')} sat-naive {r['accsat/naive'].get('gbs')} sat {r['accsat/default'].get('gbs')} frac {r['accsat/default'].get('frac')} [{r['tuned'].get('schedule')}]")
PY
