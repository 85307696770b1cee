"""Host-buffer execution with the PCIe transfers overlapped with compute.

``run_host(kernel, host_arrays, scalars)`` is ``eval_region`` for arrays that
live in (pinned) host memory in the reference layout, as a satcc user holds
them: the outermost loop is cut into chunks of planes and three CUDA streams
overlap, chunk by chunk,

    H2D of chunk c+1's planes  |  remap + kernel on chunk c  |  D2H of the planes c-1 finished

Which planes a chunk needs comes from the kernel's subscript-0 reach
(``acs_kernel_array_reach``): loaded arrays contribute [p0+ld_lo, p1+ld_hi),
stored arrays [p0+st_lo, p1+st_hi) (uploaded so elements the nest does not
write keep their host values); a stored plane is downloaded once no later
chunk can write it.  Every plane crosses PCIe exactly once per direction, so
the call approaches max(H2D bytes, D2H bytes) / link bandwidth instead of
their sum plus the compute.  Numerics are those of one whole-range launch
(each chunk is the same kernel over a sub-range of the outermost loop).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List

from . import backend


@dataclass
class Reach:
    sliced: bool
    loaded: bool
    stored: bool
    ld_lo: int
    ld_hi: int
    st_lo: int
    st_hi: int


def reaches(k: backend.Kernel) -> Dict[str, Reach]:
    L = backend.lib()
    f = L.acs_kernel_array_reach
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 7
    out = {}
    for i, name in enumerate(k.info["arrays"]):
        v = [ctypes.c_int() for _ in range(7)]
        backend._check(f(k.handle, i, *[ctypes.byref(x) for x in v]), "acs_kernel_array_reach")
        out[name] = Reach(bool(v[0].value), bool(v[1].value), bool(v[2].value), *[x.value for x in v[3:]])
    return out


class HostRunner:
    """Reusable device buffers + streams for repeated host-buffer calls of one
    kernel on one problem shape."""

    def __init__(self, k: backend.Kernel, host: Dict[str, object], range_params, chunks: int = 8):
        import torch
        self.torch = torch
        self.k = k
        self.host = host
        self.rp = range_params
        self.chunks = chunks
        self.reach = reaches(k)
        self.rm = {n: torch.empty(tuple(t.shape), dtype=t.dtype, device="cuda") for n, t in host.items()}
        self.nat = {n: backend.empty_native(k, n, tuple(t.shape), t.dtype) for n, t in host.items()}
        self.s_h2d, self.s_cmp, self.s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.launches = 0

    def _copy_planes(self, name, lo, hi, to_device, stream):
        """H2D (+ remap into the native layout) or (remap +) D2H of planes [lo, hi)."""
        t = self.host[name]
        lo, hi = max(lo, 0), min(hi, t.shape[0])
        if hi <= lo:
            return
        torch = self.torch
        with torch.cuda.stream(stream):
            if to_device:
                self.rm[name][lo:hi].copy_(t[lo:hi], non_blocking=True)
                backend.copy(self.nat[name][lo:hi], self.rm[name][lo:hi], stream)
            else:
                backend.copy(self.rm[name][lo:hi], self.nat[name][lo:hi], stream)
                t[lo:hi].copy_(self.rm[name][lo:hi], non_blocking=True)
        self.launches += 1

    def run(self, scalars: Dict[str, float], variant: str = "accsat", schedule="default") -> None:
        torch = self.torch
        beg, end = self.rp
        b, e = int(scalars[beg]), int(scalars[end])
        n = e - b
        cuts = [b + n * c // self.chunks for c in range(self.chunks + 1)]
        cur = torch.cuda.current_stream()
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        # whole (non-sliced) arrays once
        with torch.cuda.stream(self.s_h2d):
            for name, r in self.reach.items():
                if not r.sliced and (r.loaded or r.stored):
                    self.rm[name].copy_(self.host[name], non_blocking=True)
                    backend.copy(self.nat[name], self.rm[name], self.s_h2d)
        uploaded = {n: -10**9 for n in self.host}        # highest plane uploaded so far (exclusive)
        downloaded = {n: -10**9 for n in self.host}
        for name, r in self.reach.items():
            if r.sliced:
                uploaded[name] = 0 if not (r.loaded or r.stored) else -10**9
        h2d_done: List = []
        cmp_done: List = []
        for c in range(self.chunks):
            p0, p1 = cuts[c], cuts[c + 1]
            for name, r in self.reach.items():
                if not r.sliced or not (r.loaded or r.stored):
                    continue
                lo = p0 + min(r.ld_lo if r.loaded else 0, r.st_lo if r.stored else 0)
                hi = p1 + max(r.ld_hi if r.loaded else 0, r.st_hi if r.stored else 0)
                if c == 0:
                    lo = min(lo, 0)                      # planes below the loop range: copied once
                if c == self.chunks - 1:
                    hi = max(hi, self.host[name].shape[0])
                lo = max(lo, uploaded[name])
                self._copy_planes(name, lo, hi, True, self.s_h2d)
                uploaded[name] = max(uploaded[name], hi)
            ev = torch.cuda.Event()
            ev.record(self.s_h2d)
            h2d_done.append(ev)
            self.s_cmp.wait_event(ev)
            sc = dict(scalars)
            sc[beg], sc[end] = p0, p1
            self.k.launch(self.nat, sc, variant, schedule, self.s_cmp)
            self.launches += 1
            ev2 = torch.cuda.Event()
            ev2.record(self.s_cmp)
            cmp_done.append(ev2)
            # planes no later chunk writes are final
            self.s_d2h.wait_event(ev2)
            for name, r in self.reach.items():
                if not (r.sliced and r.stored):
                    continue
                if c + 1 < self.chunks:
                    final_hi = cuts[c + 1] + r.st_lo
                else:
                    final_hi = self.host[name].shape[0]
                lo = max(downloaded[name], 0 if c == 0 else downloaded[name])
                lo = 0 if c == 0 else lo
                self._copy_planes(name, lo, final_hi, False, self.s_d2h)
                downloaded[name] = max(downloaded[name], final_hi)
        # non-sliced stored arrays come back whole
        with torch.cuda.stream(self.s_d2h):
            for name, r in self.reach.items():
                if not r.sliced and r.stored:
                    backend.copy(self.rm[name], self.nat[name], self.s_d2h)
                    self.host[name].copy_(self.rm[name], non_blocking=True)
        cur.wait_stream(self.s_d2h)

    def bytes_per_call(self):
        h2d = d2h = 0
        for name, r in self.reach.items():
            t = self.host[name]
            nb = t.numel() * t.element_size()
            if r.loaded or r.stored:
                h2d += nb
            if r.stored:
                d2h += nb
        return h2d, d2h
