mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "d3q19 or stream_collide" > gpurun_out/pytest_d3q19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d3q19.log
tail -3 gpurun_out/pytest_d3q19.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-table --no-cpu --no-e2e > gpurun_out/bench_d3q19.json 2> gpurun_out/bench_d3q19.err
cat gpurun_out/bench_d3q19.json; tail -3 gpurun_out/bench_d3q19.err
