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
chunk can write it.  Every plane crosses PCIe at most once per direction, so
the call approaches max(H2D bytes, D2H bytes) / link bandwidth instead of
their sum plus the compute.

A stored array the nest never loads is uploaded only OUTSIDE its write core:
the box every launch overwrites whatever the inputs are, derived from the
kernel's unconditional store targets (``acs_kernel_must_write``) and the
iteration space (``acs_kernel_iteration_space``).  Only the shell around the
core keeps host values (D3Q19 ``dst``: 120 MB of 2.6 GB), copied as a few
strided DMA boxes (``acs_copy_box``).  Numerics are those of one whole-range launch
(each chunk is the same kernel over a sub-range of the outermost loop).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
import itertools
from typing import Dict, List, Optional, Tuple

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


def write_core(k: backend.Kernel, name: str, dims, scalars) -> Optional[List[Tuple[int, int]]]:
    """Box [lo, hi) per position that the launch overwrites for ANY input:
    every component combination of the absolute subscripts has a target, and
    the loop-mapped positions take the intersection of the shifted
    iteration ranges.  None when there is no such box."""
    loop_of, targets = k.must_write(name)
    nd = len(dims)
    space = k.iteration_space(scalars)
    if not targets or any(h <= l for l, h in space):
        return None
    lpos = [p for p in range(nd) if loop_of[p] >= 0]
    apos = [p for p in range(nd) if loop_of[p] < 0]
    if len({loop_of[p] for p in lpos}) != len(lpos):
        return None                                   # one loop in two positions: not a box
    combos = 1
    for p in apos:
        combos *= dims[p]
    if combos > 4096:
        return None
    by_combo: Dict[tuple, tuple] = {}
    for t in targets:
        by_combo.setdefault(tuple(t[p] for p in apos), t)
    core = [[0, dims[p]] for p in range(nd)]
    for c in itertools.product(*[range(dims[p]) for p in apos]):
        t = by_combo.get(tuple(c))
        if t is None:
            return None
        for p in lpos:
            lo, hi = space[loop_of[p]]
            core[p][0] = max(core[p][0], lo + t[p])
            core[p][1] = min(core[p][1], hi + t[p])
    core = [(max(0, l), min(dims[p], h)) for p, (l, h) in enumerate(core)]
    if any(h <= l for l, h in core):
        return None
    return core


def shell_boxes(dims, core) -> List[Tuple[List[int], List[int]]]:
    """The full array minus the core box, as disjoint boxes: for position p,
    positions < p inside the core, p below or above it, positions > p full."""
    out = []
    nd = len(dims)
    for p in range(nd):
        for lo_p, hi_p in ((0, core[p][0]), (core[p][1], dims[p])):
            if hi_p <= lo_p:
                continue
            lo = [core[q][0] for q in range(p)] + [lo_p] + [0] * (nd - p - 1)
            hi = [core[q][1] for q in range(p)] + [hi_p] + list(dims[p + 1:])
            out.append((lo, hi))
    return out


class HostRunner:
    """Reusable device buffers + streams for repeated host-buffer calls of one
    kernel on one problem shape."""

    def __init__(self, k: backend.Kernel, host: Dict[str, object], range_params, chunks: int = 8,
                 ramp: bool = False):
        import torch
        self.torch = torch
        self.k = k
        self.host = host
        self.rp = range_params
        self.chunks = chunks
        self.ramp = ramp
        self.reach = reaches(k)
        self.rm = {n: torch.empty(tuple(t.shape), dtype=t.dtype, device="cuda") for n, t in host.items()}
        # a 0/1 mask the nest declares `int` may be held on the host as bytes
        # (D3Q19 flags: 17 MB instead of 68 MB over PCIe per call); the device
        # copy the kernel reads is int32, widened by the remap (acs_copy u8 -> i32)
        self.nat = {n: backend.empty_native(k, n, tuple(t.shape), torch.int32 if t.dtype == torch.uint8 else t.dtype)
                    for n, t in host.items()}
        self.s_h2d, self.s_cmp, self.s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.s_d2h2 = torch.cuda.Stream()      # second download stream (a second copy engine)
        self.split_d2h = False
        self.launches = 0
        self.shell: Dict[str, List] = {}      # store-only arrays: boxes outside the write core
        self._shell_key = None

    def _cuts(self, b: int, n: int) -> List[int]:
        """Chunk boundaries of the outermost loop.  With `ramp`, the first and
        last chunks are smaller (1/4, 1/2 of the rest): the download can start
        sooner and the final download after the last kernel is shorter."""
        C = self.chunks
        if not self.ramp or C < 6:
            return [b + n * c // C for c in range(C + 1)]
        w = [1.0] * C
        w[0] = w[-1] = 0.25
        w[1] = w[-2] = 0.5
        tot = sum(w)
        cuts, acc = [b], 0.0
        for c in range(C):
            acc += w[c]
            cuts.append(b + int(round(n * acc / tot)))
        cuts[-1] = b + n
        out = [cuts[0]]
        for x in cuts[1:]:
            if x > out[-1]:
                out.append(x)
        return out

    def _plan_shells(self, scalars):
        key = tuple(sorted((n, float(v)) for n, v in scalars.items()))
        if key == self._shell_key:
            return
        self._shell_key = key
        self.shell = {}
        for name, r in self.reach.items():
            if r.sliced and r.stored and not r.loaded:
                dims = tuple(self.host[name].shape)
                core = write_core(self.k, name, dims, scalars)
                if core is not None:
                    self.shell[name] = shell_boxes(dims, core)

    def _h2d(self, name, lo, hi, stream):
        """Pinned host -> device staging (reference layout) of planes [lo, hi):
        copy engine only, so the H2D stream never waits on a kernel."""
        t = self.host[name]
        with self.torch.cuda.stream(stream):
            if name in self.shell:
                # only the part of planes [lo, hi) outside the write core
                for blo, bhi in self.shell[name]:
                    l0, h0 = max(blo[0], lo), min(bhi[0], hi)
                    if h0 > l0:
                        backend.copy_box(self.rm[name], t, [l0] + blo[1:], [h0] + bhi[1:], stream)
            else:
                self.rm[name][lo:hi].copy_(t[lo:hi], non_blocking=True)
        self.launches += 1

    @staticmethod
    def _clip(lo, hi, n):
        return max(lo, 0), min(hi, n)

    def run(self, scalars: Dict[str, float], variant: str = "accsat", schedule="default") -> None:
        """Three streams: H2D (copy engine) | remap-in + kernel + remap-out |
        D2H (copy engine), chained per chunk by events."""
        torch = self.torch
        self._plan_shells(scalars)
        beg, end = self.rp
        b, e = int(scalars[beg]), int(scalars[end])
        n = e - b
        cuts = self._cuts(b, n)
        nch = len(cuts) - 1
        cur = torch.cuda.current_stream()
        for s in (self.s_h2d, self.s_cmp, self.s_d2h, self.s_d2h2):
            s.wait_stream(cur)
        # whole (non-sliced) arrays once
        whole = [name for name, r in self.reach.items() if not r.sliced and (r.loaded or r.stored)]
        with torch.cuda.stream(self.s_h2d):
            for name in whole:
                self.rm[name].copy_(self.host[name], non_blocking=True)
        uploaded = {nm: -10**9 for nm in self.host}       # highest plane uploaded so far (exclusive)
        downloaded = {nm: -10**9 for nm in self.host}
        first = True
        for c in range(nch):
            p0, p1 = cuts[c], cuts[c + 1]
            remap_in = []
            for name, r in self.reach.items():
                if not r.sliced or not (r.loaded or r.stored):
                    continue
                lo = p0 + min(r.ld_lo if r.loaded else 0, r.st_lo if r.stored else 0)
                hi = p1 + max(r.ld_hi if r.loaded else 0, r.st_hi if r.stored else 0)
                if c == 0:
                    lo = min(lo, 0)                      # planes below the loop range: copied once
                if c == nch - 1:
                    hi = max(hi, self.host[name].shape[0])
                lo = max(lo, uploaded[name])
                lo, hi = self._clip(lo, hi, self.host[name].shape[0])
                if hi > lo:
                    self._h2d(name, lo, hi, self.s_h2d)
                    remap_in.append((name, lo, hi))
                uploaded[name] = max(uploaded[name], hi)
            ev = torch.cuda.Event()
            ev.record(self.s_h2d)
            self.s_cmp.wait_event(ev)
            if first:
                for name in whole:
                    backend.copy(self.nat[name], self.rm[name], self.s_cmp)
                first = False
            for name, lo, hi in remap_in:
                backend.copy(self.nat[name][lo:hi], self.rm[name][lo:hi], self.s_cmp)
            sc = dict(scalars)
            sc[beg], sc[end] = p0, p1
            self.k.launch(self.nat, sc, variant, schedule, self.s_cmp)
            self.launches += 1
            # planes no later chunk writes are final: remap out, then D2H
            out = []
            for name, r in self.reach.items():
                if not (r.sliced and r.stored):
                    continue
                final_hi = cuts[c + 1] + r.st_lo if c + 1 < nch else self.host[name].shape[0]
                lo = 0 if c == 0 else downloaded[name]
                lo, hi = self._clip(lo, final_hi, self.host[name].shape[0])
                if hi > lo:
                    backend.copy(self.rm[name][lo:hi], self.nat[name][lo:hi], self.s_cmp)
                    out.append((name, lo, hi))
                downloaded[name] = max(downloaded[name], final_hi)
            if c == nch - 1:
                for name, r in self.reach.items():
                    if not r.sliced and r.stored:
                        backend.copy(self.rm[name], self.nat[name], self.s_cmp)
                        out.append((name, 0, self.host[name].shape[0]))
            ev2 = torch.cuda.Event()
            ev2.record(self.s_cmp)
            self.s_d2h.wait_event(ev2)
            if self.split_d2h:
                self.s_d2h2.wait_event(ev2)
            for name, lo, hi in out:
                mid = (lo + hi) // 2 if self.split_d2h and hi - lo > 1 else hi
                with torch.cuda.stream(self.s_d2h):
                    self.host[name][lo:mid].copy_(self.rm[name][lo:mid], non_blocking=True)
                if mid < hi:
                    with torch.cuda.stream(self.s_d2h2):
                        self.host[name][mid:hi].copy_(self.rm[name][mid:hi], non_blocking=True)
                self.launches += 1
        cur.wait_stream(self.s_d2h)
        cur.wait_stream(self.s_d2h2)

    def capture(self, scalars: Dict[str, float], variant: str = "accsat", schedule="default"):
        """The whole call (every chunk's H2D, remap, launch, remap, D2H on the
        three streams) captured once as a CUDA graph; replay() re-runs it on
        the current host buffers with no per-chunk host work."""
        torch = self.torch
        self.run(scalars, variant, schedule)           # warm: plans, attributes, tensor maps
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cs):
            self.run(scalars, variant, schedule)
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        return g

    def bytes_per_call(self):
        h2d = d2h = 0
        for name, r in self.reach.items():
            t = self.host[name]
            nb = t.numel() * t.element_size()
            if name in self.shell:
                es = t.element_size()
                for lo, hi in self.shell[name]:
                    n = 1
                    for a, b in zip(lo, hi):
                        n *= b - a
                    h2d += n * es
            elif r.loaded or r.stored:
                h2d += nb
            if r.stored:
                d2h += nb
        return h2d, d2h
