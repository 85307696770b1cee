# Full default bench (both arms) on one GPU.
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
tail -n 3 gpurun_out/bench.err gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
