# ncu --set full of every nest's tuned accsat kernel, summarised on the box (reports are large).
# usage: gpurun -- bash tools/gpu/profile_all.sh
# ncu --set full of every nest's tuned accsat kernel (one launch each)
mkdir -p gpurun_out; rm -f gpurun_out/profile_slots.txt
cap() {  # name kid slot|tuned [f32]   (tuned: ask the tuner first, outside ncu)
  S=$3; [ "$S" = tuned ] && S=$(python tools/gpu/profile_kernel.py $2 accsat tuned $4 | tail -1)
  echo "$1 slot $S" >> gpurun_out/profile_slots.txt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'naive_kernel|naive_multi_kernel|march_kernel|stream_kernel|sliced_kernel' -s 1 -c 1 -o gpurun_out/r01_$1 python tools/gpu/profile_kernel.py $2 accsat $S $4 3 > gpurun_out/ncu_$1.log 2>&1
}
cap jacobi7 jacobi7.c:jacobi7:0 tuned
cap d3q19 d3q19.c:stream_collide:0 tuned
cap calc1 swim.c:calc1:0 tuned
cap calc2 swim.c:calc2:1 tuned
cap calc3 swim.c:calc3:2 tuned
cap ideal_gas clover.c:ideal_gas:0 tuned
cap pdv clover.c:pdv_predict:1 tuned
cap advec clover.c:advec_cell_x:2 tuned
cap wave4 wave4.c:wave4:0 tuned f32
cap zsolve zsolve.c:z_solve_lhs:0 tuned
ls gpurun_out/r01_*.ncu-rep | wc -l
python tools/summarize_ncu.py gpurun_out/r01_all_kernels.md gpurun_out/r01_jacobi7.ncu-rep=268435456 gpurun_out/r01_d3q19.ncu-rep=5117050880 gpurun_out/r01_calc1.ncu-rep=3758096384 gpurun_out/r01_calc2.ncu-rep=5368709120 gpurun_out/r01_calc3.ncu-rep=8053063680 gpurun_out/r01_ideal_gas.ncu-rep=1887436800 gpurun_out/r01_pdv.ncu-rep=5662310400 gpurun_out/r01_advec.ncu-rep=2831155200 gpurun_out/r01_wave4.ncu-rep=17179869184 gpurun_out/r01_zsolve.ncu-rep=16777216000 > gpurun_out/summ.log 2>&1
cp profiles/traffic.json gpurun_out/traffic_box.json
for f in gpurun_out/r01_*.ncu-rep; do case $f in *d3q19*) ;; *) rm -f $f ;; esac; done
du -sh gpurun_out
