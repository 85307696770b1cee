mkdir -p gpurun_out
export ACS_DEBUG=1
C="python tools/gpu/check_case.py"
timeout 200 compute-sanitizer --tool memcheck $C d3q19.c:stream_collide:0 "(5,6,35)" accsat > gpurun_out/dbg3.log 2>&1
timeout 120 $C jacobi7.c:jacobi7:0 "(9,47,20)" original > gpurun_out/dbg2.log 2>&1
timeout 120 $C clover.c:advec_cell_x:2 "(131,257)" accsat >> gpurun_out/dbg2.log 2>&1
timeout 120 $C wave4.c:wave4:0 "(19,22,61)" accsat tiled f32 >> gpurun_out/dbg2.log 2>&1
timeout 120 $C swim.c:calc1:0 "(131,257)" accsat >> gpurun_out/dbg2.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not stream_collide and not d3q19" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
