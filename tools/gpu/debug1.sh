mkdir -p gpurun_out
export ACS_DEBUG=1
C="python tools/gpu/check_case.py"
timeout 120 $C jacobi7.c:jacobi7:0 "(9,9,70)" original > gpurun_out/dbg2.log 2>&1
timeout 120 $C jacobi7.c:jacobi7:0 "(9,47,20)" original >> gpurun_out/dbg2.log 2>&1
timeout 120 $C jacobi7.c:jacobi7:0 "(33,9,20)" original >> gpurun_out/dbg2.log 2>&1
timeout 120 $C d3q19.c:stream_collide:0 "(13,17,35)" accsat >> gpurun_out/dbg2.log 2>&1
timeout 120 $C clover.c:pdv_predict:1 "(131,257)" accsat >> gpurun_out/dbg2.log 2>&1
timeout 120 $C clover.c:advec_cell_x:2 "(131,257)" accsat >> gpurun_out/dbg2.log 2>&1
timeout 120 $C wave4.c:wave4:0 "(19,22,61)" accsat tiled f32 >> gpurun_out/dbg2.log 2>&1
timeout 200 compute-sanitizer --tool memcheck $C jacobi7.c:jacobi7:0 "(33,47,70)" original > gpurun_out/dbg1.log 2>&1
echo done
