mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_tab.json 2> gpurun_out/bench_tab.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_tab.json'))
for k,r in d['per_kernel'].items():
    print(f"{k:14s} orig {r['original/naive'].get('gbs')} nvcc {r['original-nvcc/naive'].get('gbs')} sat {r['accsat/default'].get('gbs')} frac {r['accsat/default'].get('frac')} x{r.get('sat_vs_orig_speedup')} xnvcc {r.get('sat_vs_nvcc_default_speedup')}")
PY
timeout 900 ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_st.sum,smsp__inst_executed_op_shared_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum -k regex:'naive_kernel|march_kernel|stream_kernel|sliced_kernel' --csv --log-file gpurun_out/inst_metrics.csv python tools/gpu/inst_evidence.py gpurun_out/inst_plan.json > gpurun_out/inst.log 2>&1
tail -2 gpurun_out/inst.log
