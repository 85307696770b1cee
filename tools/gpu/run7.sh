mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_shard.py -q -p no:cacheprovider -x > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
tail -3 gpurun_out/pytest_shard.log
P="python tools/gpu/profile_kernel.py"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 -o gpurun_out/prof_advec_march $P clover.c:advec_cell_x:2 accsat 17 f64 3 > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 2 -c 1 -o gpurun_out/prof_jacobi_march4 $P jacobi7.c:jacobi7:0 accsat 20 f64 3 > gpurun_out/ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:naive_kernel -s 2 -c 1 -o gpurun_out/prof_d3q19_naive3 $P d3q19.c:stream_collide:0 accsat 17 f64 3 > gpurun_out/ncu3.log 2>&1
echo done
