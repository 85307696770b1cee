# Round check on one GPU: every GPU test (sanitizer included), smoke, every bench line,
# the ncu launch list of the default bench and --set full captures of the headline kernels.
# usage: gpurun -- bash tools/gpu/round_check.sh
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu/bench_all.sh > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-table --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
W4=$(python tools/gpu/profile_kernel.py wave4.c:wave4:0 accsat tuned f32 2>/dev/null | tail -1)
bash tools/gpu/prof_one.sh wave4_r02 wave4.c:wave4:0 $W4 f32 > /dev/null 2>&1
J=$(python tools/gpu/profile_kernel.py jacobi7.c:jacobi7:0 accsat tuned 2>/dev/null | tail -1)
bash tools/gpu/prof_one.sh jacobi_r02 jacobi7.c:jacobi7:0 $J > /dev/null 2>&1
echo "wave4 slot $W4 jacobi slot $J" > gpurun_out/prof_slots.txt
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/prof_slots.txt
echo done
