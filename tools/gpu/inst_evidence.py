#!/usr/bin/env python3
"""Launch sequence for the instruction / global-load evidence table: every
nest at a mid size, once per (variant, schedule) in a fixed order, so an ncu
metrics pass over this process maps launch i -> row i of the printed plan.

   ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_op_global_ld.sum,\
smsp__inst_executed_op_global_st.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
gpu__time_duration.sum -k regex:'naive_kernel|march_kernel|stream_kernel' --csv \
       python tools/gpu/inst_evidence.py plan.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2306_13002_b200 import backend, nests  # noqa: E402

SIZES = {"jacobi7": 256, "d3q19": 128, "swim": 4096, "clover": 4096, "wave4": 512, "zsolve": 128}
plan = []
for kid, spec in nests.KERNELS.items():
    dtype = "f32" if spec.nest == "wave4" else "f64"
    w = nests.workload(kid, SIZES[spec.nest], dtype=dtype)
    k = backend.Kernel.lookup(kid)
    arrs = nests.device_inputs(w, native=True, kernel=k)
    for variant, sched in (("original", "naive"), ("original-nvcc", "naive"), ("accsat", "naive"), ("accsat", "tiled")):
        k.launch(arrs, dict(w.scalars), variant, sched)
        torch.cuda.synchronize()
        prec = 1 if dtype == "f32" else 0
        slot = 0 if sched == "naive" else "tiled"
        plan.append({"kernel": kid, "variant": variant, "schedule": sched, "points": w.points,
                     "algorithmic_bytes": w.algorithmic_bytes, "dtype": dtype,
                     "static_loads": k.info["static_loads"][0 if variant.startswith("original") else 4],
                     "fma": k.info["fma_count"][0 if variant.startswith("original") else 4]})
    del arrs
    torch.cuda.empty_cache()
with open(sys.argv[1] if len(sys.argv) > 1 else "plan.json", "w") as f:
    json.dump(plan, f, indent=1)
print("launches", len(plan))
