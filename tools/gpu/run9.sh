mkdir -p gpurun_out
timeout 900 ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_st.sum,smsp__inst_executed_op_shared_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum -k regex:'naive_kernel|march_kernel|stream_kernel' --csv --log-file gpurun_out/inst_metrics.csv python tools/gpu/inst_evidence.py gpurun_out/inst_plan.json > gpurun_out/inst.log 2>&1
ACS_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --size 128 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "n2 rc=$?" >> gpurun_out/bench_n2.err
echo done
