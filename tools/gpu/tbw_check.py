"""wave4 temporal-blocking check on one GPU: fp32 1024^3, 12 time steps per timed step —
the tuned single-step kernel (12 launches, rotation) vs acs_launch_leapfrog2 (6 launches,
4-buffer rotation), interleaved reps, median ms per time step and GB/s of the algorithmic
bytes (16 B/point/step).  usage: python tools/gpu/tbw_check.py [reps] [size]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2306_13002_b200 import backend, nests  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 9
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
kid = "wave4.c:wave4:0"
w = nests.workload(kid, size, dtype="f32")
k = backend.Kernel.lookup(kid)
arrs = nests.device_inputs(w, native=True, kernel=k)
x = torch.empty_like(arrs["un"])
x = backend.empty_native(k, "un", tuple(arrs["un"].shape), arrs["un"].dtype)
sc = dict(w.scalars)
best, tms = k.tune(arrs, sc, "accsat", reps=5)
STEPS = 12


def single():
    b = dict(arrs)
    for t in range(STEPS):
        roles = nests.role_buffers("wave4", ["u", "up", "un", "vel2"], t)
        k.launch({p: arrs[r] for p, r in roles.items()}, sc, "accsat")


def blocked():
    bufs = {"u": arrs["u"], "up": arrs["up"], "un": arrs["un"], "x": x}
    for _ in range(STEPS // 2):
        k.launch_leapfrog2({"u": bufs["u"], "up": bufs["up"], "un": bufs["un"], "vel2": arrs["vel2"]}, bufs["x"],
                           sc, "accsat")
        bufs = {"u": bufs["x"], "up": bufs["un"], "un": bufs["up"], "x": bufs["u"]}


fns = {"single": single, "tb2": blocked}
for f in fns.values():
    f()
torch.cuda.synchronize()
ev = {n: [] for n in fns}
for _ in range(reps):
    for n, f in fns.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        ev[n].append((a, b))
torch.cuda.synchronize()
out = {"size": size, "tuned_slot": best}
for n in fns:
    ms = sorted(a.elapsed_time(b) / STEPS for a, b in ev[n])
    med = statistics.median(ms)
    out[n] = {"ms_per_step": round(med, 4), "iqr": round(ms[3 * len(ms) // 4] - ms[len(ms) // 4], 4),
              "gbs": round(w.algorithmic_bytes / (med * 1e-3) / 1e9, 1)}
out["speedup"] = round(out["single"]["ms_per_step"] / out["tb2"]["ms_per_step"], 3)
print(json.dumps(out))
