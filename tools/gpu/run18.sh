mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sliced_kernel -s 1 -c 1 -o gpurun_out/prof_zsolve_sliced python tools/gpu/profile_kernel.py zsolve.c:z_solve_lhs:0 accsat 17 > gpurun_out/ncu_zs.log 2>&1
tail -3 gpurun_out/ncu_zs.log
