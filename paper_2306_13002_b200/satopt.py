"""Python front-end of host stage (a) — libacs_opt.so (include/accsat_opt.h).

    text, metrics = satopt.optimize_source(source, "swim.c", "accsat")

mirrors the reference's optimize_source (proj/include/satcc/pipeline.hpp:64-66):
emitted module text plus satcc-metrics-v1 region metrics."""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libacs_opt.so")
CLI_PATH = os.path.join(HERE, "acs-satcc")


class Limits(ctypes.Structure):
    _fields_ = [("max_nodes", ctypes.c_long), ("max_time_s", ctypes.c_double), ("max_iters", ctypes.c_int),
                ("dag_search", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.acs_opt_optimize.restype = ctypes.c_int
        L.acs_opt_optimize.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(Limits),
                                       ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
        L.acs_opt_verify.restype = ctypes.c_int
        L.acs_opt_verify.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(Limits),
                                     ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_void_p)]
        L.acs_opt_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def optimize_source(source: str, name: str = "<input>", variant: str = "accsat", max_nodes: int = 10000,
                    max_time_s: float = 10.0, max_iters: int = 10, dag_search: bool = True) -> Tuple[str, dict]:
    lim = Limits(max_nodes, max_time_s, max_iters, 1 if dag_search else 0)
    t, j = ctypes.c_void_p(), ctypes.c_void_p()
    rc = lib().acs_opt_optimize(source.encode(), name.encode(), variant.encode(), ctypes.byref(lim),
                                ctypes.byref(t), ctypes.byref(j))
    text = ctypes.string_at(t).decode()
    meta = json.loads(ctypes.string_at(j).decode())
    lib().acs_opt_free(t)
    lib().acs_opt_free(j)
    if rc != 0:
        raise SyntaxError(meta.get("error", "parse failure"))
    return text, meta


def verify_source(source: str, name: str = "<input>", variant: str = "accsat", trials: int = 20,
                  tol_rel: float = 1e-6, max_nodes: int = 10000, max_time_s: float = 10.0, max_iters: int = 10,
                  dag_search: bool = True) -> Tuple[bool, dict]:
    """satcc verify for one source: (all regions ok, per-file report)."""
    lim = Limits(max_nodes, max_time_s, max_iters, 1 if dag_search else 0)
    j = ctypes.c_void_p()
    rc = lib().acs_opt_verify(source.encode(), name.encode(), variant.encode(), ctypes.byref(lim), trials, tol_rel,
                              ctypes.byref(j))
    rep = json.loads(ctypes.string_at(j).decode())
    lib().acs_opt_free(j)
    if rc == 2:
        raise SyntaxError(rep.get("error", "parse failure"))
    return rc == 0, rep

