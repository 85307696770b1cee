# one wave4 two-step configuration: parity, interleaved timing (3 runs)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k leapfrog2 -x > gpurun_out/tbw_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc $(tail -1 gpurun_out/tbw_pytest.log)"; [ $rc -eq 0 ] || exit 1
for r in 1 2 3; do timeout 300 python tools/gpu/tbw_check.py 7 2>/dev/null; done
