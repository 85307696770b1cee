# Temporal-blocking configuration x k-chunk sweep (Jacobi-7 256^3, 100 sweeps), after parity of
# the new configurations.  usage: gpurun -- bash tools/gpu/tb2_sweep.sh "<cfgs>" "<kchunks>"
mkdir -p gpurun_out
CFGS=${1:-"0 3 4"}; KCS=${2:-"0 20 28 40"}
for cfg in $CFGS; do
  ACS_TB_CFG=$cfg timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k temporal -x > gpurun_out/tb2_pytest_$cfg.log 2>&1
  rc=$?; echo "cfg $cfg pytest rc=$rc $(tail -1 gpurun_out/tb2_pytest_$cfg.log)"
  [ $rc -eq 0 ] || exit 1
done
for rep in 1 2; do
for cfg in $CFGS; do for kc in $KCS; do
  if [ $kc = 0 ]; then unset ACS_TB_KCHUNK; else export ACS_TB_KCHUNK=$kc; fi
  ACS_TB_CFG=$cfg timeout 300 python tools/gpu/tb2_check.py 7 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg kchunk $kc', d['tb2']['ms'], d['tb2']['iqr_ms'], d['single']['ms'], d['speedup'])"
done; done; done | tee gpurun_out/tb2_sweep.txt
