# wave4 two-step kernel: k-chunk sweep and one ncu --set full capture.  usage: gpurun -- bash tools/gpu/tbw_prof.sh
mkdir -p gpurun_out
for kc in 0 64 128 256; do
  if [ $kc = 0 ]; then unset ACS_TB_KCHUNK; else export ACS_TB_KCHUNK=$kc; fi
  timeout 300 python tools/gpu/tbw_check.py 5 2>/dev/null | sed "s/^/kchunk $kc: /"
done | tee gpurun_out/tbw_sweep.txt
unset ACS_TB_KCHUNK
ACS_TB_KCHUNK=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tbw_kernel -s 1 -c 1 -o gpurun_out/tbw -f \
  python tools/gpu/tbw_check.py 1 > gpurun_out/tbw_ncu.log 2>&1; echo "ncu rc=$?"
