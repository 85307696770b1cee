"""Host-side mirror of the reference's execution API over the C ABI.

``eval_region`` here is the drop-in for the reference's

    Environment eval_region(const Stmt& body, Environment env)
        (proj/include/satcc/interp.hpp:72-74, proj/src/interp.cpp:266-270)

with the same value semantics — the environment is copied in and a new one
returned — except that it executes the WHOLE nest of one registered region on
the B200 (libaccsat_b200.so, include/accsat_b200.h) instead of tree-walking
it.  Errors map to the reference's exception types: ``EvalError`` for
runtime failures (bounds, missing names — proj/include/satcc/diag.hpp:43-47),
``InternalError`` for broken invariants (diag.hpp:50-53).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libaccsat_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "accsat_b200.h")

ACS_OK, ACS_E_ARG, ACS_E_NO_KERNEL, ACS_E_SHAPE, ACS_E_CUDA, ACS_E_NCCL, ACS_E_BOUNDS, ACS_E_LAYOUT = range(8)
F64, F32, I32, I64, U8 = range(5)
VARIANTS = {"original": 0, "cse": 1, "cse+bulk": 2, "cse+sat": 3, "accsat": 4,
            "original-nvcc": 5}   # measurement baseline: original text, nvcc-default arithmetic
SCHEDULES = {"default": 0, "naive": 1, "tiled": 2}
FILL = {"uniform": 0, "const": 1, "mask": 2, "d3q19": 3}
MAX_DIMS = 8


class EvalError(RuntimeError):
    """Runtime failure of a nest (satcc::EvalError analogue)."""


class InternalError(RuntimeError):
    """Broken invariant / backend failure (satcc::InternalError analogue)."""


class AcsArray(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("dtype", ctypes.c_int), ("ndim", ctypes.c_int32),
                ("dims", ctypes.c_int64 * MAX_DIMS), ("strides", ctypes.c_int64 * MAX_DIMS),
                ("data", ctypes.c_void_p)]


class AcsScalar(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("is_int", ctypes.c_int32), ("i", ctypes.c_int64),
                ("d", ctypes.c_double)]


class AcsKernelInfo(ctypes.Structure):
    _fields_ = [("kernel_id", ctypes.c_char_p), ("function", ctypes.c_char_p), ("region", ctypes.c_int32),
                ("n_loops", ctypes.c_int32), ("n_arrays", ctypes.c_int32), ("n_scalars", ctypes.c_int32),
                ("static_loads", ctypes.c_int32 * 5), ("fma_count", ctypes.c_int32 * 5),
                ("has_tiled", ctypes.c_int32), ("has_f32", ctypes.c_int32), ("n_schedules", ctypes.c_int32)]


EXPORTS = {
    "acs_abi_version": (ctypes.c_int, []),
    "acs_last_error": (ctypes.c_char_p, []),
    "acs_kernel_count": (ctypes.c_int, []),
    "acs_kernel_id": (ctypes.c_char_p, [ctypes.c_int]),
    "acs_lookup": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "acs_kernel_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(AcsKernelInfo)]),
    "acs_kernel_array_name": (ctypes.c_char_p, [ctypes.c_void_p, ctypes.c_int]),
    "acs_kernel_scalar_name": (ctypes.c_char_p, [ctypes.c_void_p, ctypes.c_int]),
    "acs_kernel_scalar_is_int": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "acs_launch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(AcsArray),
                                  ctypes.c_int, ctypes.POINTER(AcsScalar), ctypes.c_int, ctypes.c_void_p]),
    "acs_kernel_schedule_name": (ctypes.c_char_p, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "acs_tune": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(AcsArray), ctypes.c_int,
                                ctypes.POINTER(AcsScalar), ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_float)]),
    "acs_fill": (ctypes.c_int, [ctypes.POINTER(AcsArray), ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p]),
    "acs_copy": (ctypes.c_int, [ctypes.POINTER(AcsArray), ctypes.POINTER(AcsArray), ctypes.c_void_p]),
    "acs_native_strides": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
}

_lib = None


def lib():
    """The loaded backend.  Raises if the sm_100a library was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise InternalError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, what: str) -> None:
    if status == ACS_OK:
        return
    msg = lib().acs_last_error().decode()
    if status in (ACS_E_BOUNDS, ACS_E_ARG, ACS_E_SHAPE, ACS_E_NO_KERNEL, ACS_E_LAYOUT):
        raise EvalError(f"{what}: {msg}")
    raise InternalError(f"{what}: {msg}")


def kernel_ids():
    L = lib()
    return [L.acs_kernel_id(i).decode() for i in range(L.acs_kernel_count())]


# ---------------------------------------------------------------------------
# tensors <-> descriptors (torch is used for device memory and streams only)

def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    m = {torch.float64: F64, torch.float32: F32, torch.int32: I32, torch.int64: I64, torch.uint8: U8}
    return m[t.dtype]


def describe(name: str, t) -> AcsArray:
    """acs_array for a torch CUDA tensor (any strides)."""
    a = AcsArray()
    a.name = name.encode()
    a.dtype = _dtype_code(t)
    a.ndim = t.dim()
    for p in range(t.dim()):
        a.dims[p] = t.shape[p]
        a.strides[p] = t.stride(p)
    a.data = t.data_ptr()
    return a


def _stream_handle(stream) -> Optional[int]:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class Kernel:
    """One registered region (a C-ABI acs_kernel handle)."""
    kernel_id: str
    handle: int
    info: Dict = field(default_factory=dict)

    @classmethod
    def lookup(cls, kernel_id: str) -> "Kernel":
        h = ctypes.c_void_p()
        _check(lib().acs_lookup(kernel_id.encode(), ctypes.byref(h)), "acs_lookup")
        inf = AcsKernelInfo()
        _check(lib().acs_kernel_get_info(h, ctypes.byref(inf)), "acs_kernel_get_info")
        info = {"function": inf.function.decode(), "region": inf.region, "n_loops": inf.n_loops,
                "static_loads": list(inf.static_loads), "fma_count": list(inf.fma_count),
                "has_tiled": bool(inf.has_tiled), "has_f32": bool(inf.has_f32),
                "n_schedules": inf.n_schedules,
                "schedules": [[(lib().acs_kernel_schedule_name(h, prec, i) or b"").decode() for i in range(8)]
                              for prec in (0, 1)],
                "arrays": [lib().acs_kernel_array_name(h, i).decode() for i in range(inf.n_arrays)],
                "scalars": [lib().acs_kernel_scalar_name(h, i).decode() for i in range(inf.n_scalars)],
                "scalar_is_int": [lib().acs_kernel_scalar_is_int(h, i) for i in range(inf.n_scalars)]}
        return cls(kernel_id, h.value, info)

    @staticmethod
    def _pack(arrays, scalars):
        descs = (AcsArray * len(arrays))(*[describe(n, t) for n, t in arrays.items()])
        sc = (AcsScalar * len(scalars))()
        for i, (n, v) in enumerate(scalars.items()):
            sc[i].name = n.encode()
            is_int = isinstance(v, (int, np.integer)) and not isinstance(v, bool)
            sc[i].is_int = 1 if is_int else 0
            sc[i].i = int(v) if is_int else 0
            sc[i].d = float(v)
        return descs, sc

    def launch(self, arrays: Dict[str, object], scalars: Dict[str, float], variant: str = "accsat",
               schedule="default", stream=None) -> None:
        """Asynchronous launch on `stream` (torch stream; default current).
        `schedule`: "default" | "naive" | "tiled" | int slot (0 = naive)."""
        descs, sc = self._pack(arrays, scalars)
        sched = 16 + schedule if isinstance(schedule, int) else SCHEDULES[schedule]
        _check(lib().acs_launch(self.handle, VARIANTS[variant], sched, descs, len(arrays), sc,
                                len(scalars), _stream_handle(stream)), f"acs_launch({self.kernel_id}, {variant})")

    def launch_steps(self, arrays: Dict[str, object], scalars: Dict[str, float], variant: str = "accsat",
                     nsteps: int = 1, blocked: bool = True, stream=None) -> str:
        """acs_launch_steps: `nsteps` steps of a ping-pong nest's time loop
        (two per launch with temporal blocking where registered); returns the
        name of the array holding the newest field."""
        names = list(arrays)
        descs, sc = self._pack(arrays, scalars)
        latest = ctypes.c_int(-1)
        f = lib().acs_launch_steps
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(AcsArray), ctypes.c_int, ctypes.POINTER(AcsScalar),
                      ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
        _check(f(self.handle, VARIANTS[variant], descs, len(names), sc, len(scalars), nsteps, 1 if blocked else 0,
                 _stream_handle(stream), ctypes.byref(latest)), f"acs_launch_steps({self.kernel_id})")
        return names[latest.value]

    def launch_leapfrog2(self, arrays: Dict[str, object], un2, scalars: Dict[str, float], variant: str = "accsat",
                         stream=None) -> None:
        """acs_launch_leapfrog2: two steps of a 3-level leapfrog nest (wave4) in
        one launch: step 1 into arrays["un"], step 2 into `un2` (a fourth buffer
        of un's layout).  Afterwards the time loop's up is un, its u is un2."""
        descs, sc = self._pack(arrays, scalars)
        extra = describe("un2", un2)
        f = lib().acs_launch_leapfrog2
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(AcsArray), ctypes.c_int, ctypes.POINTER(AcsScalar),
                      ctypes.c_int, ctypes.POINTER(AcsArray), ctypes.c_void_p]
        _check(f(self.handle, VARIANTS[variant], descs, len(arrays), sc, len(scalars), ctypes.byref(extra),
                 _stream_handle(stream)), f"acs_launch_leapfrog2({self.kernel_id}, {variant})")

    def tune(self, arrays, scalars, variant: str = "accsat", reps: int = 3, stream=None):
        """acs_tune: times every registered schedule slot on these arrays and
        makes the fastest the default for this variant.  Returns
        (best_slot, {slot: ms})."""
        descs, sc = self._pack(arrays, scalars)
        best = ctypes.c_int(-1)
        ms = (ctypes.c_float * 8)()
        _check(lib().acs_tune(self.handle, VARIANTS[variant], descs, len(arrays), sc, len(scalars),
                              _stream_handle(stream), reps, ctypes.byref(best), ms), f"acs_tune({self.kernel_id})")
        return best.value, {i: ms[i] for i in range(8) if ms[i] >= 0}

    def iteration_space(self, scalars: Dict[str, float]) -> List[Tuple[int, int]]:
        """[lo, hi) of every marked loop (outermost first) for these scalars."""
        _, sc = self._pack({}, scalars)
        n = self.info["n_loops"]
        lo, hi = (ctypes.c_int64 * 8)(), (ctypes.c_int64 * 8)()
        f = lib().acs_kernel_iteration_space
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _check(f(self.handle, sc, len(scalars), lo, hi), "acs_kernel_iteration_space")
        return [(lo[d], hi[d]) for d in range(n)]

    def must_write(self, name: str) -> Tuple[List[int], List[Tuple[int, ...]]]:
        """(loop index or -1 per subscript position, unconditional store targets)."""
        idx = self.info["arrays"].index(name)
        loop_of = (ctypes.c_int32 * 8)()
        n = ctypes.c_int()
        f = lib().acs_kernel_must_write
        f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _check(f(self.handle, idx, loop_of, 0, None, ctypes.byref(n)), "acs_kernel_must_write")
        offs = (ctypes.c_int32 * (8 * max(1, n.value)))()
        _check(f(self.handle, idx, loop_of, n.value, offs, ctypes.byref(n)), "acs_kernel_must_write")
        return list(loop_of), [tuple(offs[i * 8:(i + 1) * 8]) for i in range(n.value)]

    def native_strides(self, name: str, dims: Tuple[int, ...]) -> Tuple[int, ...]:
        d = (ctypes.c_int64 * len(dims))(*dims)
        s = (ctypes.c_int64 * len(dims))()
        _check(lib().acs_native_strides(self.handle, name.encode(), len(dims), d, s), "acs_native_strides")
        return tuple(s)


def fill(t, kind: str, seed: int, lo: float = 0.0, hi: float = 1.0, p: float = 0.0, stream=None,
         flat_offset: int = 0) -> None:
    """acs_fill; `flat_offset` = reference flat index of t's first element
    within a larger (global) array, so a slab reproduces its share."""
    a = describe("fill", t)
    _check(lib().acs_fill(ctypes.byref(a), FILL[kind], seed, lo, hi, p, flat_offset, _stream_handle(stream)),
           "acs_fill")


def copy_box(dst, src, lo, hi, stream=None) -> None:
    """acs_copy_box: box [lo, hi) of two row-major tensors with equal shapes
    (host<->device, async on `stream`; pinned host memory overlaps)."""
    assert tuple(dst.shape) == tuple(src.shape) and dst.dtype == src.dtype
    assert dst.is_contiguous() and src.is_contiguous()
    nd = dst.dim()
    kind = {(False, True): 0, (True, False): 1, (True, True): 2}.get((src.is_cuda, dst.is_cuda), 3)
    f = lib().acs_copy_box
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    dims = (ctypes.c_int64 * nd)(*dst.shape)
    l, h = (ctypes.c_int64 * nd)(*lo), (ctypes.c_int64 * nd)(*hi)
    _check(f(dst.data_ptr(), src.data_ptr(), dst.element_size(), nd, dims, l, h, kind, _stream_handle(stream)),
           "acs_copy_box")


def copy(dst, src, stream=None) -> None:
    a, b = describe("dst", dst), describe("src", src)
    _check(lib().acs_copy(ctypes.byref(a), ctypes.byref(b), _stream_handle(stream)), "acs_copy")


def native_offset(kernel: Kernel, name: str, esize: int) -> int:
    off = ctypes.c_int64()
    f = lib().acs_native_offset
    f.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p]
    _check(f(kernel.handle, name.encode(), esize, ctypes.byref(off)), "acs_native_offset")
    return off.value


def empty_native(kernel: Kernel, name: str, dims, dtype, device="cuda", shared_with=()):
    """Device tensor with the backend's preferred strides and start offset for
    `name` (acs_native_strides / acs_native_offset).  `shared_with`: other
    kernels that read the same array; when their preferred start offsets
    differ the array starts 16-byte aligned (every skeleton takes that)."""
    torch = _torch()
    st = kernel.native_strides(name, tuple(dims))
    n = int(np.prod(dims))
    if not n:
        return torch.empty(tuple(dims), dtype=dtype, device=device)
    esize = torch.empty((), dtype=dtype).element_size()
    off = ctypes.c_int64(native_offset(kernel, name, esize))
    if any(native_offset(k, name, esize) != off.value for k in shared_with):
        off = ctypes.c_int64(0)
    if off.value == 0:
        return torch.empty_strided(tuple(dims), st, dtype=dtype, device=device)
    span = 1 + sum((d - 1) * s for d, s in zip(dims, st))
    flat = torch.empty(off.value + span, dtype=dtype, device=device)
    return flat.as_strided(tuple(dims), st, off.value)


# ---------------------------------------------------------------------------
# Environment / eval_region mirror

@dataclass
class Environment:
    """Name-keyed state (satcc::Environment, proj/include/satcc/interp.hpp:51-54):
    host numpy arrays (reference row-major layout) and Python scalars."""
    scalars: Dict[str, float] = field(default_factory=dict)
    arrays: Dict[str, np.ndarray] = field(default_factory=dict)

    def copy(self) -> "Environment":
        return Environment(dict(self.scalars), {k: v.copy() for k, v in self.arrays.items()})


_NP2TORCH = None


def _to_device(a: np.ndarray, kernel: Kernel, name: str, native: bool):
    torch = _torch()
    host = torch.from_numpy(np.ascontiguousarray(a))
    if not native:
        return host.to("cuda", non_blocking=False)
    dev_rm = host.to("cuda")
    st = kernel.native_strides(name, tuple(a.shape))
    rm = tuple(dev_rm.stride())
    if st == rm:
        return dev_rm
    dev = torch.empty_strided(tuple(a.shape), st, dtype=dev_rm.dtype, device="cuda")
    copy(dev, dev_rm)
    return dev


def eval_region(kernel_id: str, env: Environment, variant: str = "accsat", schedule: str = "default",
                native_layout: bool = True) -> Environment:
    """Runs the whole nest of `kernel_id` on the B200 over a copy of `env`
    and returns the post-state (value semantics, like satcc::eval_region)."""
    torch = _torch()
    if not torch.cuda.is_available():
        raise InternalError("no CUDA device visible: the B200 backend has no CPU fallback")
    k = Kernel.lookup(kernel_id)
    dev = {}
    for name in k.info["arrays"]:
        if name not in env.arrays:
            raise EvalError(f"read of undefined array: {name}")
        dev[name] = _to_device(env.arrays[name], k, name, native_layout)
    sc = {}
    for name, is_int in zip(k.info["scalars"], k.info["scalar_is_int"]):
        if name not in env.scalars:
            raise EvalError(f"read of undefined variable: {name}")
        v = env.scalars[name]
        sc[name] = int(v) if is_int else float(v)
    k.launch(dev, sc, variant, schedule)
    out = env.copy()
    for name, t in dev.items():
        if t.is_contiguous():
            out.arrays[name] = t.cpu().numpy()
        else:
            rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
            copy(rm, t)
            out.arrays[name] = rm.cpu().numpy()
    torch.cuda.synchronize()
    return out
