#!/usr/bin/env python3
"""Runs one nest at its BASELINE size a few times (for ncu captures):
   python tools/gpu/profile_kernel.py <kernel_id> <variant> <schedule|tuned> [f32] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2306_13002_b200 import backend, nests  # noqa: E402

kid, variant, sched = sys.argv[1], sys.argv[2], sys.argv[3]
sched = int(sched) - 16 if sched.isdigit() and int(sched) >= 16 else (int(sched) if sched.isdigit() else sched)
dtype = "f32" if len(sys.argv) > 4 and sys.argv[4] == "f32" else "f64"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
w = nests.workload(kid, None, dtype=dtype)
k = backend.Kernel.lookup(kid)
arrs = nests.device_inputs(w, native=True, kernel=k)
if sched == "tuned":                       # print the tuner's choice (as a profile_kernel slot) and exit
    best, _ = k.tune(arrs, dict(w.scalars), variant)
    print(best + 16 if best > 0 else "naive")
    sys.exit(0)
torch.cuda.synchronize()
for _ in range(reps):
    k.launch(arrs, dict(w.scalars), variant, sched)
torch.cuda.synchronize()
print("ok", kid, variant, sched, dtype)
