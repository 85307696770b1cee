"""Temporal blocking check on one GPU: Jacobi-7 256^3, 100 sweeps per step —
the single-sweep tuned graph vs acs_launch_steps with two sweeps per launch
(kernels/tblock.cuh).  Interleaved reps, median ms and GB/s of the algorithmic
bytes (16 B/point/sweep).  usage: python tools/gpu/tb2_check.py [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
kid = "jacobi7.c:jacobi7:0"
slot, name, _ = bench.tune_kernel(kid, 256, "f64", "accsat")
res, w = bench.bench_configs(kid, 256, "f64", 100, [("accsat", slot), ("accsat", "tb2")], reps)
out = {"tuned_slot": slot, "tuned": name, "single": res[0], "tb2": res[1],
       "speedup": round(res[0]["ms"] / res[1]["ms"], 3)}
print(json.dumps(out))
