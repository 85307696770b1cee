"""ctypes front-end of the CPU oracle (oracle/_ref/libacs_cpu.so).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path.

The library holds, for every nest function F and form:
  F__original        the nest text (nests/<nest>.c)            gcc -O3 -ffp-contract=off
  F__cse|cse_bulk|cse_sat|accsat
                     host stage (a)'s emitted text for that VariantConfig
                     (paper_2306_13002_b200/emitted/ — the program the GPU
                     kernels are lowered from), two-rounding FMA as the
                     reference interpreter evaluates it (proj/src/interp.cpp:68-70)
  F__ref_<form>      the same for the REFERENCE optimizer's emitted text
                     (tests/golden/emitted/), the cross-check
  F__cse_sat_fma|accsat_fma
                     the same text with each extracted FMA as one fma() —
                     the arithmetic the sm_100a saturated kernels perform
  …_f32              (wave4) the textual fp32 copy
and an ``_omp`` twin of each that splits the outermost loop over threads.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libacs_cpu.so")

FORM_OF_VARIANT = {"original": "original", "cse": "cse", "cse+bulk": "cse_bulk",
                   "cse+sat": "cse_sat", "accsat": "accsat"}

_lib = None


def build() -> str:
    import sys
    subprocess.run([sys.executable, os.path.join(HERE, "gen_oracle_c.py")], check=True, stdout=subprocess.DEVNULL)
    subprocess.run(["make", "-s", "-C", HERE, "cpu"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def form_name(variant: str, fma: bool = False, f32: bool = False, ref: bool = False) -> str:
    f = FORM_OF_VARIANT[variant]
    if ref and variant != "original":
        f = "ref_" + f
    if fma and variant in ("cse+sat", "accsat"):
        f += "_fma"
    if f32:
        f += "_f32"
    return f


def run(spec, arrays: Dict[str, np.ndarray], scalars: Dict[str, float], variant: str = "original",
        fma: bool = False, f32: bool = False, threads: int = 0, ref: bool = False) -> None:
    """Runs one nest function IN PLACE on host arrays (reference layout).

    `spec` is a nests.KernelSpec; `threads` > 0 uses the OpenMP driver;
    `ref` runs the reference optimizer's emitted text for `variant` instead of
    host stage (a)'s."""
    n = len(spec.params)
    a = (ctypes.c_void_p * n)()
    d = (ctypes.c_long * (8 * n))()
    iv = (ctypes.c_longlong * n)()
    dv = (ctypes.c_double * n)()
    for p in spec.params:
        if p.dims:
            arr = arrays[p.name]
            assert arr.flags["C_CONTIGUOUS"], p.name
            a[p.position] = arr.ctypes.data
            for k, v in enumerate(arr.shape):
                d[8 * p.position + k] = v
        elif p.ctype == "int":
            iv[p.position] = int(scalars[p.name])
        else:
            dv[p.position] = float(scalars[p.name])
    sym = f"{spec.function}__{form_name(variant, fma, f32, ref)}"
    if threads > 0:
        fn = getattr(lib(), sym + "_omp")
        fn.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int]
        fn(a, d, iv, dv, threads)
    else:
        fn = getattr(lib(), sym)
        fn.argtypes = [ctypes.c_void_p] * 4
        fn(a, d, iv, dv)


_FILL_KIND = {"uniform": 0, "const": 1, "mask": 2, "d3q19": 3}


def host_inputs(w, threads: int = 0) -> Dict[str, np.ndarray]:
    """Reference-layout host inputs of a nests.Workload, filled in place by
    oracle/fill.c (OpenMP) — bit-identical to nests.make_inputs, without its
    full-size numpy temporaries.  For bench.py's reference arm."""
    import os as _os
    from paper_2306_13002_b200 import nests
    f = lib().acs_cpu_fill
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                  ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
    threads = threads or _os.cpu_count() or 1
    fdt = np.float32 if w.dtype == "f32" else np.float64
    out: Dict[str, np.ndarray] = {}
    for p in w.spec.arrays:
        shape = w.dims[p.name]
        fl = w.fills[p.name]
        dt = np.int32 if p.ctype == "int" else fdt
        if fl.kind == "copy":
            out[p.name] = out[fl.src].copy()
            continue
        a = np.empty(shape, dtype=dt)
        code = 2 if dt == np.int32 else (1 if dt == np.float32 else 0)
        lo = fl.value if fl.kind == "const" else fl.lo
        if f(a.ctypes.data, a.size, code, _FILL_KIND[fl.kind], nests.SEED_BASE + p.position, lo, fl.hi, fl.p, 0,
             threads):
            raise RuntimeError(f"acs_cpu_fill failed for {p.name}")
        out[p.name] = a
    return out
