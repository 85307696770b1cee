# Temporal-blocking iteration on one GPU: parity (two sweeps per launch vs step by step) for every
# registered configuration (ACS_TB_CFG), timing against the tuned single-sweep graph, one
# ncu --set full capture of the default configuration.
# usage: gpurun -- bash tools/gpu/tb2_iter.sh
mkdir -p gpurun_out
for cfg in 0 1 2; do
  ACS_TB_CFG=$cfg timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k temporal -x > gpurun_out/tb2_pytest_$cfg.log 2>&1
  rc=$?; echo "cfg $cfg pytest rc=$rc"; tail -1 gpurun_out/tb2_pytest_$cfg.log
  [ $rc -eq 0 ] || exit 1
done
for cfg in 0 1 2 0 1 2; do
  ACS_TB_CFG=$cfg timeout 300 python tools/gpu/tb2_check.py 9 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg', d['tb2'], d['single'], d['speedup'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb2_kernel -s 2 -c 1 -o gpurun_out/tb2 -f \
  python tools/gpu/tb2_check.py 2 > gpurun_out/tb2_ncu.log 2>&1; echo "ncu rc=$?"
