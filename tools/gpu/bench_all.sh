# Every bench line on one GPU: default (wave4 1024^3, per-kernel table, e2e, cpu baseline),
# the reference arm, the other workloads (D3Q19, swim and CloverLeaf steps) with their
# reference arms, and the N=2 torchrun path time-sharing the one GPU (functional only).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
for w in d3q19 swim clover; do
  timeout 900 python bench.py --workload $w --no-table > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "rc=$?" >> gpurun_out/bench_$w.err
  timeout 900 python bench.py --workload $w --impl reference > gpurun_out/bench_ref_$w.json 2> gpurun_out/bench_ref_$w.err; echo "rc=$?" >> gpurun_out/bench_ref_$w.err
done
for w in wave4 swim; do
  ACS_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --workload $w --no-table --no-cpu --steps 6 --warmup 3 > gpurun_out/bench_n2_$w.json 2> gpurun_out/bench_n2_$w.err; echo "rc=$?" >> gpurun_out/bench_n2_$w.err
done
tail -n 2 gpurun_out/*.err
