python tools/gpu/graph_probe.py > gpurun_out/graph_probe.json 2>&1; cat gpurun_out/graph_probe.json
