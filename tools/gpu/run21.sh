mkdir -p gpurun_out
for s in 20 21; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 1 -c 1 -o gpurun_out/prof_jac_$s python tools/gpu/profile_kernel.py jacobi7.c:jacobi7:0 accsat $s > gpurun_out/ncu_jac$s.log 2>&1
done
for s in 20 21; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 1 -c 1 -o gpurun_out/prof_w4_$s python tools/gpu/profile_kernel.py wave4.c:wave4:0 accsat $s f32 > gpurun_out/ncu_w4$s.log 2>&1
done
