# ncu --set full of the D3Q19 tuned kernel (slot 1), summarised on the box
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:naive_kernel -s 1 -c 1 -o gpurun_out/r01_d3q19_off python tools/gpu/profile_kernel.py d3q19.c:stream_collide:0 accsat 17 3 > gpurun_out/ncu_d3q19_off.log 2>&1
python tools/summarize_ncu.py gpurun_out/r01_d3q19_off.md gpurun_out/r01_d3q19_off.ncu-rep=5117050880 > /dev/null 2>&1
cat gpurun_out/r01_d3q19_off.md | grep -E "Duration|DRAM|Occupancy|stalls|Issue"
