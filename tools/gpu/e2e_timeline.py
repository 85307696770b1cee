"""Per-stream busy timeline of one e2e D3Q19 call (torch profiler / CUPTI):
when each H2D, kernel and D2H ran, to see where the call loses time against
the PCIe floor."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2306_13002_b200 import backend, nests, pipeline_exec  # noqa: E402

kid = "d3q19.c:stream_collide:0"
w = nests.workload(kid, 256)
k = backend.Kernel.lookup(kid)
dev = nests.device_inputs(w, native=False, kernel=k)
host = {n: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for n, t in dev.items()}
for n, t in dev.items():
    host[n].copy_(t)
del dev
torch.cuda.synchronize()
r = pipeline_exec.HostRunner(k, host, w.spec.range_params, chunks=16)
sc = dict(w.scalars)
r.run(sc)
r.run(sc)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.run(sc)
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type.name == "CUDA":
        evs.append((e.time_range.start, e.time_range.end, e.name[:60]))
evs.sort()
t0 = evs[0][0]
kinds = {}
for s, e, n in evs:
    key = "memcpy HtoD" if "HtoD" in n else ("memcpy DtoH" if "DtoH" in n else ("remap" if "copy" in n.lower() or "remap" in n.lower() else "kernel" if "kernel" in n else n))
    d = kinds.setdefault(key, {"n": 0, "busy_ms": 0.0, "first_ms": 1e9, "last_ms": 0.0})
    d["n"] += 1
    d["busy_ms"] += (e - s) / 1e3
    d["first_ms"] = min(d["first_ms"], (s - t0) / 1e3)
    d["last_ms"] = max(d["last_ms"], (e - t0) / 1e3)
print(json.dumps({"span_ms": (max(e for _, e, _ in evs) - t0) / 1e3, "by_kind": kinds}, indent=1))
print("\n".join(f"{(s - t0) / 1e3:8.2f} {(e - s) / 1e3:7.2f}  {n}" for s, e, n in evs[:60]))
