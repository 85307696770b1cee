"""satcc-metrics-v1 with GPU fields (SURVEY.md §5 "metrics / logging").

``acs-satcc report --gpu [--size N] file.c ...`` (or ``python -m
paper_2306_13002_b200.report ...``) prints the reference CLI's per-region
metrics (``metrics_json``, proj/tools/satcc_main.cpp:89-110: objective and
static loads before/after, FMAs, method, ...) from host stage (a), and adds
to every region the B200 execution of the same form:

  "gpu": {"kernel_id", "grid", "dtype", "schedule" (the slot acs_tune picked),
          "ms" (median launch), "gbs", "roofline_frac" (of the measured HBM
          copy peak), "bytes_per_point", "static_loads" / "fma_count" of the
          registered kernel, "vs_original": {max_abs, max_rel, bitwise} —
          the saturated form against the original form, both on the GPU, on
          the same inputs (the diff_test of proj/src/oracle.cpp:64-81 applied
          to whole nests)}

Regions of files that are not registered benchmark nests report
``"gpu": {"error": ...}`` (``acs-satcc --backend b200`` runs those).
"""
from __future__ import annotations

import json
import os
import sys
from typing import Dict, List, Optional

import numpy as np

from . import backend, nests, satopt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def gpu_fields(kid: str, variant: str = "accsat", size=None, reps: int = 10) -> Dict:
    import torch
    spec = nests.kernel(kid)
    dtype = "f32" if spec.nest == "wave4" else "f64"
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    arrs = nests.device_inputs(w, native=True, kernel=k)
    slot, _ = k.tune(arrs, dict(w.scalars), variant, reps=5)
    prec = 1 if dtype == "f32" else 0
    stream = torch.cuda.current_stream()
    outs = {}
    for v in (variant, "original"):
        arrs = nests.device_inputs(w, native=True, kernel=k)          # same seeded inputs for both forms
        k.launch(arrs, dict(w.scalars), v, "default", stream)
        torch.cuda.synchronize()
        outs[v] = {n: _to_host(arrs[n]) for n in w.write_arrays}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for i in range(reps):
        k.launch(arrs, dict(w.scalars), variant, "default", stream)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]))
    max_abs = max_rel = 0.0
    bitwise = True
    for n in w.write_arrays:
        a, b = outs[variant][n].astype(np.float64), outs["original"][n].astype(np.float64)
        d = np.abs(a - b)
        bitwise &= bool(np.array_equal(outs[variant][n], outs["original"][n]))
        max_abs = max(max_abs, float(d.max(initial=0.0)))
        mag = np.maximum(np.abs(a), np.abs(b))
        with np.errstate(invalid="ignore", divide="ignore"):
            rel = np.where(mag > 0, d / mag, 0.0)
        max_rel = max(max_rel, float(rel.max(initial=0.0)))
    del arrs
    torch.cuda.empty_cache()
    gbs = w.algorithmic_bytes / (ms * 1e-3) / 1e9
    vi = ["original", "cse", "cse+bulk", "cse+sat", "accsat"].index(variant)
    return {"kernel_id": kid, "grid": [int(d) for d in w.dims[w.spec.arrays[0].name]], "dtype": dtype,
            "schedule": k.info["schedules"][prec][slot], "ms": round(ms, 4), "gbs": round(gbs, 1),
            "roofline_frac": round(gbs / _peak(), 4), "peak_gbs": _peak(), "bytes_per_point": w.bytes_per_point,
            "static_loads": k.info["static_loads"][vi], "fma_count": k.info["fma_count"][vi],
            "vs_original": {"max_abs": max_abs, "max_rel": max_rel, "bitwise": bitwise}}


def _to_host(t):
    import torch
    if not t.is_contiguous():
        rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
        backend.copy(rm, t)
        t = rm
    return t.cpu().numpy()


def report(path: str, variant: str = "accsat", gpu: bool = True, size=None) -> Dict:
    src = open(path).read()
    name = os.path.basename(path)
    _, meta = satopt.optimize_source(src, path, variant, exact_time_s=satopt.EXACT_TIME_S)
    if gpu:
        registered = set(backend.kernel_ids())
        for r in meta["regions"]:
            kid = f"{name}:{r['function']}:{r['region']}"
            if kid not in registered:
                r["gpu"] = {"error": f"{kid} is not a registered kernel (acs-satcc --backend b200 runs it)"}
                continue
            try:
                r["gpu"] = gpu_fields(kid, variant, size)
            except Exception as e:   # report, never hide
                r["gpu"] = {"error": str(e)[:300]}
    return meta


def main(argv: List[str]) -> int:
    variant, gpu, size, files = "accsat", False, None, []
    args = list(argv)
    while args:
        a = args.pop(0)
        if a == "--variant":
            variant = args.pop(0)
        elif a == "--gpu":
            gpu = True
        elif a == "--size":
            size = int(args.pop(0))
        else:
            files.append(a)
    if not files:
        print("usage: python -m paper_2306_13002_b200.report [--gpu] [--size N] [--variant V] file.c ...",
              file=sys.stderr)
        return 2
    print(json.dumps([report(f, variant, gpu, size) for f in files], indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
