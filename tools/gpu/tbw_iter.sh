# wave4 temporal-blocking iteration: parity (two fp32 steps per launch vs step by step), then timing
# against the tuned single-step kernel (tools/gpu/tbw_check.py).  usage: gpurun -- bash tools/gpu/tbw_iter.sh
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k leapfrog2 -x > gpurun_out/tbw_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc"; tail -3 gpurun_out/tbw_pytest.log
[ $rc -eq 0 ] || exit 1
timeout 900 python tools/gpu/tbw_check.py 9 > gpurun_out/tbw_check.json 2> gpurun_out/tbw_check.err; echo "check rc=$?"
cat gpurun_out/tbw_check.json; tail -3 gpurun_out/tbw_check.err
