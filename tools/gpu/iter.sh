# Iteration check on one GPU: shard tests, ABI tests, bench (short), reference arm.
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_abi.py -q -x -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_shard.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-table > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
tail -3 gpurun_out/pytest_shard.log; cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -n 3 gpurun_out/bench.err gpurun_out/bench_ref.err
