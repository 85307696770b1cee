# tb2 x-shuffle variant (ACS_TB_CFG=5) vs the default: parity, interleaved timing, ncu of the variant.
mkdir -p gpurun_out
ACS_TB_CFG=5 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k temporal -x > gpurun_out/tb2_pytest_5.log 2>&1
rc=$?; echo "cfg 5 pytest rc=$rc $(tail -1 gpurun_out/tb2_pytest_5.log)"; [ $rc -eq 0 ] || exit 1
for rep in 1 2 3; do for cfg in 0 5; do
  ACS_TB_CFG=$cfg timeout 300 python tools/gpu/tb2_check.py 9 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg', d['tb2']['ms'], d['tb2']['iqr_ms'], d['single']['ms'], d['speedup'])"
done; done | tee gpurun_out/tb2_xs.txt
ACS_TB_CFG=5 timeout 900 ncu --set full --clock-control none -k regex:tb2_kernel -s 2 -c 1 -o gpurun_out/tb2_xs -f \
  python tools/gpu/tb2_check.py 2 > gpurun_out/tb2_xs_ncu.log 2>&1; echo "ncu rc=$?"
