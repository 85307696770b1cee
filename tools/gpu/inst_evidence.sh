# Instruction / global-load evidence (ncu metrics over tools/gpu/inst_evidence.py), then
# python tools/inst_table.py gpurun_out/inst_plan.json gpurun_out/inst_metrics.csv
mkdir -p gpurun_out
timeout 900 ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_st.sum,smsp__inst_executed_op_shared_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum -k regex:'naive_kernel|naive_multi_kernel|march_kernel|stream_kernel|sliced_kernel' --csv --log-file gpurun_out/inst_metrics.csv python tools/gpu/inst_evidence.py gpurun_out/inst_plan.json > gpurun_out/inst.log 2>&1
tail -2 gpurun_out/inst.log
