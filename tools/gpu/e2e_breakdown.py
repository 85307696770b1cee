"""Where the e2e (host-buffer) D3Q19 step spends its time: H2D stream alone,
shell boxes alone, D2H alone, and the full overlapped call."""
import json
import os
import sys

import torch

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
chunks = int(os.environ.get("CHUNKS", "16"))
r = pipeline_exec.HostRunner(k, host, w.spec.range_params, chunks=chunks)
sc = dict(w.scalars)
r.run(sc)
torch.cuda.synchronize()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


s = torch.cuda.current_stream()
res = {}
for rnd in range(2):
    res[f"full_ms_{rnd}"] = timed(lambda: r.run(sc), reps=5)
    res[f"h2d_src_ms_{rnd}"] = timed(lambda: r.rm["src"].copy_(host["src"], non_blocking=True), reps=5)
    res[f"h2d_dst_whole_ms_{rnd}"] = timed(lambda: r.rm["dst"].copy_(host["dst"], non_blocking=True), reps=5)
res["full_ms"] = timed(lambda: r.run(sc))
res["h2d_src_ms"] = timed(lambda: r.rm["src"].copy_(host["src"], non_blocking=True))
res["h2d_flags_ms"] = timed(lambda: r.rm["flags"].copy_(host["flags"], non_blocking=True))
res["h2d_dst_shell_ms"] = timed(lambda: r._h2d("dst", 0, 258, s))
res["h2d_dst_whole_ms"] = timed(lambda: r.rm["dst"].copy_(host["dst"], non_blocking=True))
res["d2h_dst_ms"] = timed(lambda: host["dst"].copy_(r.rm["dst"], non_blocking=True))
res["kernel_ms"] = timed(lambda: k.launch(r.nat, sc, "accsat", "default", s))
res["remap_src_ms"] = timed(lambda: backend.copy(r.nat["src"], r.rm["src"], s))
res["shell_boxes"] = [(lo, hi) for lo, hi in r.shell.get("dst", [])]
print(json.dumps(res))
