# the default bench line only.  usage: gpurun -- bash tools/gpu/bench_only.sh
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
