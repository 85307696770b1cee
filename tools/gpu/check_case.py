#!/usr/bin/env python3
"""One parity case through the C ABI vs the CPU oracle (debug helper):
   python tools/gpu/check_case.py <kernel_id> "<size>" <variant> [schedule] [f32]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import cpu as oracle_cpu  # noqa: E402
from test_gpu_parity import bitwise_equal, run_gpu  # noqa: E402
from paper_2306_13002_b200 import nests  # noqa: E402

kid, size, variant = sys.argv[1], eval(sys.argv[2]), sys.argv[3]
sched = sys.argv[4] if len(sys.argv) > 4 else "tiled"
f32 = len(sys.argv) > 5 and sys.argv[5] == "f32"
w = nests.workload(kid, size, dtype="f32" if f32 else "f64")
ins = nests.make_inputs(w)
want = {n: a.copy() for n, a in ins.items()}
oracle_cpu.run(w.spec, want, w.scalars, variant, fma=variant in ("accsat", "cse+sat"), f32=f32)
got = run_gpu(kid, ins, w.scalars, variant, sched)
for n in w.write_arrays:
    ok = bitwise_equal(got[n], want[n])
    bad = np.argwhere(got[n] != want[n])
    print(kid, size, variant, sched, n, "bitwise", ok, "ndiff", len(bad), bad[:5].tolist())
