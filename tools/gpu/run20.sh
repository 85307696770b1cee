mkdir -p gpurun_out
for s in 19 20; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 1 -c 1 -o gpurun_out/prof_wave4_s$s python tools/gpu/profile_kernel.py wave4.c:wave4:0 accsat $s f32 > gpurun_out/ncu_w$s.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 1 -c 1 -o gpurun_out/prof_jacobi_s21 python tools/gpu/profile_kernel.py jacobi7.c:jacobi7:0 accsat 21 > gpurun_out/ncu_j21.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 1 -c 1 -o gpurun_out/prof_jacobi_s20 python tools/gpu/profile_kernel.py jacobi7.c:jacobi7:0 accsat 20 > gpurun_out/ncu_j20.log 2>&1
ls gpurun_out/*.ncu-rep
