# Temporal-blocking iteration on one GPU: parity (two sweeps per launch vs step by step),
# timing against the tuned single-sweep graph, one ncu --set full capture of the tb2 kernel.
# usage: gpurun -- bash tools/gpu/tb2_iter.sh
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k temporal -x > gpurun_out/tb2_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc" >> gpurun_out/tb2_pytest.log; tail -3 gpurun_out/tb2_pytest.log
[ $rc -eq 0 ] || exit 1
timeout 600 python tools/gpu/tb2_check.py 15 > gpurun_out/tb2_check.json 2> gpurun_out/tb2_check.err; echo "check rc=$?"
cat gpurun_out/tb2_check.json
for kc in 16 24 32 48 64; do
  ACS_TB_KCHUNK=$kc timeout 300 python tools/gpu/tb2_check.py 7 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kchunk $kc', d['tb2'], d['single'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb2_kernel -s 2 -c 1 -o gpurun_out/tb2 -f \
  python tools/gpu/tb2_check.py 2 > gpurun_out/tb2_ncu.log 2>&1; echo "ncu rc=$?"
