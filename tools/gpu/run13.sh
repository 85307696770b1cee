mkdir -p gpurun_out
python tools/gpu/pcie_bw.py > gpurun_out/pcie.json 2>&1; cat gpurun_out/pcie.json
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "host_runner or abi" > gpurun_out/pytest_hr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hr.log
tail -3 gpurun_out/pytest_hr.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-table --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['value'],d['e2e'])"; tail -3 gpurun_out/bench_e2e.err
