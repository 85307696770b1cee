#!/usr/bin/env python3
"""Times every registered slot of one nest at its BASELINE size as the bench
does (Stepper, graph-captured multi-sweep steps, interleaved reps):
   python tools/gpu/slot_sweep.py <kernel_id> [variant] [sweeps] [reps] [f32]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2306_13002_b200 import backend  # noqa: E402

kid = sys.argv[1]
variant = sys.argv[2] if len(sys.argv) > 2 else "accsat"
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
dtype = "f32" if len(sys.argv) > 5 and sys.argv[5] == "f32" else "f64"
size = dict((k, s) for k, s, _, _ in bench.TABLE)[kid]
k = backend.Kernel.lookup(kid)
names = k.info["schedules"][1 if dtype == "f32" else 0]
slots = [i for i, n in enumerate(names) if n]
res, w = bench.bench_configs(kid, size, dtype, sweeps, [(variant, s) for s in slots], reps)
peak, _ = bench.load_peaks()
for s, r in zip(slots, res):
    print(json.dumps({"kid": kid, "slot": s, "schedule": names[s], "ms": r["ms"], "iqr": r["iqr_ms"],
                      "gbs": r["gbs"], "frac": round(r["gbs"] / peak, 4)}))
