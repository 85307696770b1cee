#!/usr/bin/env python3
"""D3Q19 layout / schedule experiment: GB/s for every schedule slot under
three layouts (q-major SoA padded = native, SoA unpadded, reference AoS)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2306_13002_b200 import backend, nests  # noqa: E402

kid = "d3q19.c:stream_collide:0"
w = nests.workload(kid, 256)
k = backend.Kernel.lookup(kid)


def alloc(layout):
    out = {}
    for p in w.spec.arrays:
        dims = w.dims[p.name]
        dt = torch.int32 if p.ctype == "int" else torch.float64
        if layout == "aos" or p.name == "flags":
            st = None
            if layout != "aos" and p.name == "flags":
                st = k.native_strides(p.name, dims) if layout == "soa_pad" else None
            t = torch.empty_strided(dims, st, dtype=dt, device="cuda") if st else torch.empty(dims, dtype=dt, device="cuda")
        elif layout == "soa_pad":
            t = backend.empty_native(k, p.name, dims, dt)
        else:  # soa, unpadded
            nz, ny, nx, q = dims
            t = torch.empty((q, nz, ny, nx), dtype=dt, device="cuda").permute(1, 2, 3, 0)
        fl = w.fills[p.name]
        backend.fill(t, fl.kind, nests.SEED_BASE + p.position, fl.lo, fl.hi, fl.p)
        out[p.name] = t
    return out


res = {}
for layout in ("soa_pad", "soa", "aos"):
    arrs = alloc(layout)
    best, ms = k.tune(arrs, dict(w.scalars), "accsat", reps=5)
    res[layout] = {k.info["schedules"][0][s]: round(w.algorithmic_bytes / (m * 1e-3) / 1e9, 1) for s, m in ms.items()}
    del arrs
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
