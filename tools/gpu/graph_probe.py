"""Host launch cost vs GPU time for the 100-sweep Jacobi step: eager ctypes
launches, and the same 100 launches captured once in a CUDA graph."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2306_13002_b200 import backend, nests  # noqa: E402

kid = "jacobi7.c:jacobi7:0"
w = nests.workload(kid, 256)
k = backend.Kernel.lookup(kid)
arrs = nests.device_inputs(w, native=True, kernel=k)
sc = dict(w.scalars)
k.tune(arrs, sc, "accsat", reps=3)
s = torch.cuda.Stream()
A, B = arrs["A0"], arrs["Anext"]


def sweeps(n=100):
    for i in range(n):
        a = {"A0": A, "Anext": B} if i % 2 == 0 else {"A0": B, "Anext": A}
        k.launch(a, sc, "accsat", "default", s)


res = {}
with torch.cuda.stream(s):
    sweeps(4)
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s):
    sweeps()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
res["eager_host_ms"] = (t1 - t0) * 1e3
res["eager_wall_ms"] = (t2 - t0) * 1e3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
with torch.cuda.stream(s):
    sweeps()
e1.record(s)
torch.cuda.synchronize()
res["eager_gpu_ms"] = e0.elapsed_time(e1)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    sweeps()
torch.cuda.synchronize()
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0.record(s)
    with torch.cuda.stream(s):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
res["graph_gpu_ms"] = best
res["graph_gbs"] = w.algorithmic_bytes * 100 / (best * 1e-3) / 1e9
print(json.dumps(res))
