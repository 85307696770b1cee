#!/usr/bin/env python3
"""Cost of the sharded step on ONE GPU: wave4 1024^3 fp32 as 1 slab (plain
launch) vs 2 and 4 slabs on the same device (peer write-through between
slabs, device flags, graph-replayed steps, every slab on its own stream).
The total work is identical, so the ratio is the sharding overhead the
kernel pays (write-through stores + wait/signal), not a scaling number."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2306_13002_b200 import shard  # noqa: E402

kid, size, steps = "wave4.c:wave4:0", (1024, 1024, 1024), 12
out = {}
for n in (1, 2, 4):
    ranks = [shard.SlabRank(kid, size, n, r, dtype="f32", schedule=2) for r in range(n)]
    for r, sr in enumerate(ranks):
        sr.connect_local(ranks[r - 1] if r > 0 else None, ranks[r + 1] if r < n - 1 else None)
    streams = [torch.cuda.Stream() for _ in ranks]
    for sr, st in zip(ranks, streams):
        sr.capture(st)
    for _ in range(3):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for _ in range(steps):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    out[n] = round(e0.elapsed_time(e1) / steps, 4)
    for sr in ranks:
        sr.close()
    del ranks
    torch.cuda.empty_cache()
print(json.dumps({"ms_per_step": out, "overhead_vs_1": {k: round(v / out[1], 4) for k, v in out.items()}}))
