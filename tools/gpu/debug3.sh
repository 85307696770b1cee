mkdir -p gpurun_out
export ACS_DEBUG=1
C="python tools/gpu/check_case.py"
timeout 200 compute-sanitizer --tool memcheck $C swim.c:calc2:1 "12" original > gpurun_out/dbg4.log 2>&1
timeout 200 compute-sanitizer --tool memcheck $C wave4.c:wave4:0 "(5,4,7)" accsat tiled f32 > gpurun_out/dbg5.log 2>&1
timeout 200 $C clover.c:advec_cell_x:2 "12" accsat > gpurun_out/dbg6.log 2>&1
timeout 200 $C clover.c:ideal_gas:0 "12" accsat >> gpurun_out/dbg6.log 2>&1
timeout 200 $C swim.c:calc3:2 "12" accsat >> gpurun_out/dbg6.log 2>&1
timeout 200 $C clover.c:pdv_predict:1 "12" accsat >> gpurun_out/dbg6.log 2>&1
echo done
