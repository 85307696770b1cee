# wave4 two-step kernel after hoisting: parity, interleaved timing (3 runs), one ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "leapfrog2 or temporal" -x > gpurun_out/tbw_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc $(tail -1 gpurun_out/tbw_pytest.log)"; [ $rc -eq 0 ] || exit 1
for r in 1 2 3; do timeout 300 python tools/gpu/tbw_check.py 7 2>/dev/null; done | tee gpurun_out/tbw_check2.txt
timeout 900 ncu --set full --clock-control none -k regex:tbw_kernel -s 1 -c 1 -o gpurun_out/tbw2 -f \
  python tools/gpu/tbw_check.py 1 > gpurun_out/tbw2_ncu.log 2>&1; echo "ncu rc=$?"
