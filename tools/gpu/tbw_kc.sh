# wave4 two-step kernel: k-chunk sweep (interleaved with the tuned single step in each run)
for kc in 64 80 96 64 80 96; do ACS_TB_KCHUNK=$kc timeout 300 python tools/gpu/tbw_check.py 5 2>/dev/null | sed "s/^/kchunk $kc: /"; done | tee gpurun_out/tbw_kc.txt
