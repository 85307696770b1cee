# ncu --set full of zsolve's tuned accsat kernel + its original's; usage: gpurun -- bash tools/gpu/prof_zsolve.sh
mkdir -p gpurun_out
Z=$(python tools/gpu/profile_kernel.py zsolve.c:z_solve_lhs:0 accsat tuned 2>/dev/null | tail -1)
echo "zsolve slot $Z"
bash tools/gpu/prof_one.sh zsolve_r02 zsolve.c:z_solve_lhs:0 $Z > /dev/null 2>&1
python tools/ncu_brief.py gpurun_out/one_zsolve_r02.ncu-rep
ncu -i gpurun_out/one_zsolve_r02.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h,v=r[0],r[2]
for k in ['smsp__inst_executed_op_global_st.sum','smsp__inst_executed_op_global_ld.sum','smsp__sass_inst_executed_op_global_st.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum','l1tex__t_requests_pipe_lsu_mem_global_op_st.sum','lts__t_sectors_srcunit_tex_op_write.sum','dram__bytes_write.sum','dram__bytes_read.sum','launch__grid_size','launch__block_size','sm__warps_active.avg.pct_of_peak_sustained_active']:
  if k in h: print(k, v[h.index(k)])
"
