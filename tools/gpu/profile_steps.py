#!/usr/bin/env python3
"""Runs acs_launch_steps (temporal blocking) on the Jacobi BASELINE grid (for ncu):
   python tools/gpu/profile_steps.py [nsteps] [variant]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2306_13002_b200 import backend, nests  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
variant = sys.argv[2] if len(sys.argv) > 2 else "accsat"
kid = "jacobi7.c:jacobi7:0"
w = nests.workload(kid, 256)
k = backend.Kernel.lookup(kid)
arrs = nests.device_inputs(w, native=True, kernel=k)
print(k.launch_steps(arrs, dict(w.scalars), variant, n, True))
torch.cuda.synchronize()
