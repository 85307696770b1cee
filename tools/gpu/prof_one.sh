# ncu --set full of one kernel: bash tools/gpu/prof_one.sh <name> <kernel_id> <slot+16> [f32]
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'naive_kernel|naive_multi_kernel|march_kernel|stream_kernel|sliced_kernel' -s 1 -c 1 -o gpurun_out/one_$1 python tools/gpu/profile_kernel.py $2 accsat $3 $4 3 > gpurun_out/ncu_one_$1.log 2>&1
ncu -i gpurun_out/one_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/one_$1_sass.csv 2>/dev/null
ls -la gpurun_out/one_$1*
