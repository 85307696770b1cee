python tools/gpu/e2e_timeline.py > gpurun_out/e2e_timeline.txt 2>&1; head -80 gpurun_out/e2e_timeline.txt
