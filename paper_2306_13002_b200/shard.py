"""Slab decomposition of a nest across GPUs.

Every benchmark nest is an independent per-point update with a bounded
stencil, so the outermost loop (k for 3-D nests, the row loop for 2-D ones)
is split into contiguous slabs, one per rank.  Each rank allocates its arrays
with the slab's planes plus the halo planes the stencil reaches, and

* computes only the planes it OWNS (local loop bounds);
* writes every store of a produced array THROUGH to the neighbour that holds
  the same global plane — from inside the compute kernel, into the
  neighbour's buffer mapped over NVLink (CUDA IPC) or on the same device
  (``acs_launch_sharded``).  wave4: the new boundary planes of ``un`` land in
  the neighbours' halos; jacobi7: ``Anext``; D3Q19: pushes into a ghost plane
  land in the owner's interior;
* orders steps across ranks with device-side release/acquire flags
  (``acs_signal`` / ``acs_wait``): step s starts only after both neighbours
  finished step s-1, so neither a halo read nor a forwarded write can race.

There is no separate exchange kernel and no host round trip per step.  The
reference has no multi-GPU path; parity is "sharded result == single-domain
result", bit for bit.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import backend, nests

# the arrays each nest produces, and how buffers rotate between steps
ROTATIONS = {
    "jacobi7": [("A0", "Anext")],
    "d3q19": [("src", "dst")],
    "wave4": [("up", "u", "un")],
}


@dataclass(frozen=True)
class SlabPlan:
    """Split of the global outermost-loop range [glo, ghi) over `nranks`.

    reach_lo / reach_hi: how far below / above its own plane any access of
    the nest goes along the sliced subscript (the array halo planes); halo:
    how far beyond its owned planes the next step READS produced data."""
    glo: int
    ghi: int
    nranks: int
    reach_lo: int
    reach_hi: int
    halo: int

    def owned(self, rank: int) -> Tuple[int, int]:
        n = self.ghi - self.glo
        lo = self.glo + n * rank // self.nranks
        hi = self.glo + n * (rank + 1) // self.nranks
        return lo, hi

    def origin(self, rank: int) -> int:
        """Global coordinate of local index 0 of this rank's buffers."""
        return self.owned(rank)[0] - self.reach_lo

    def local_planes(self, rank: int) -> int:
        lo, hi = self.owned(rank)
        return (hi - lo) + self.reach_lo + self.reach_hi

    def local_range(self, rank: int) -> Tuple[int, int]:
        """Owned planes in local coordinates (the rank's loop bounds)."""
        lo, hi = self.owned(rank)
        o = self.origin(rank)
        return lo - o, hi - o


def plan_for(w: nests.Workload, nranks: int) -> SlabPlan:
    """SlabPlan of a workload: reaches from the nest's array dims / loop
    bounds (the nests pad every array by the stencil reach), read halo from
    the stencil's load offsets along the sliced subscript."""
    beg, end = w.spec.range_params
    glo, ghi = int(w.scalars[beg]), int(w.scalars[end])
    first = next(a for a in w.spec.arrays if len(w.dims[a.name]) >= 2)
    dim0 = w.dims[first.name][0]
    reach_lo, reach_hi = glo, dim0 - ghi
    halo = {"jacobi7": 1, "wave4": 2, "d3q19": 0, "swim": 1, "clover": 1}[w.spec.nest]
    return SlabPlan(glo, ghi, nranks, reach_lo, reach_hi, halo)


def local_workload(w: nests.Workload, plan: SlabPlan, rank: int) -> nests.Workload:
    """The rank's slab of a global workload: same arrays with dims[0] cut to
    the local planes, loop bounds in local coordinates."""
    beg, end = w.spec.range_params
    dims = {}
    for a in w.spec.arrays:
        d = w.dims[a.name]
        dims[a.name] = (plan.local_planes(rank),) + tuple(d[1:]) if len(d) >= 2 else d
    lo, hi = plan.local_range(rank)
    sc = dict(w.scalars)
    sc[beg], sc[end] = lo, hi
    pts = w.points * (hi - lo) // max(1, plan.ghi - plan.glo)
    return nests.Workload(w.spec, dims, sc, w.fills, w.dtype, pts, w.bytes_per_point,
                          w.read_arrays, w.write_arrays)


def role_buffers(nest: str, names: Sequence[str], step: int) -> Dict[str, str]:
    """Parameter name -> physical buffer name at `step` (0-based)."""
    out = {n: n for n in names}
    for group in ROTATIONS.get(nest, []):
        L = len(group)
        for i, p in enumerate(group):
            out[p] = group[(i + step) % L]
    return out


# ---------------------------------------------------------------------------
# device side

class AcsShard(ctypes.Structure):
    _fields_ = [("own_lo", ctypes.c_int64), ("own_hi", ctypes.c_int64), ("origin", ctypes.c_int64),
                ("halo", ctypes.c_int32), ("n_sharded", ctypes.c_int32),
                ("names", ctypes.c_char_p * 16), ("lo_data", ctypes.c_void_p * 16),
                ("hi_data", ctypes.c_void_p * 16), ("lo_origin", ctypes.c_int64), ("hi_origin", ctypes.c_int64)]


def _fns():
    L = backend.lib()
    if not getattr(L, "_acs_shard_init", False):
        L.acs_launch_sharded.restype = ctypes.c_int
        L.acs_launch_sharded.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(backend.AcsArray),
                                         ctypes.c_int, ctypes.POINTER(backend.AcsScalar), ctypes.c_int,
                                         ctypes.POINTER(AcsShard), ctypes.c_void_p]
        L.acs_signal.restype = ctypes.c_int
        L.acs_signal.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.acs_wait.restype = ctypes.c_int
        L.acs_wait.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        L.acs_ipc_export.restype = ctypes.c_int
        L.acs_ipc_export.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        L.acs_ipc_import.restype = ctypes.c_int
        L.acs_ipc_import.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]
        L.acs_ipc_close.restype = ctypes.c_int
        L.acs_ipc_close.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L._acs_shard_init = True
    return L


def ipc_export(t) -> Tuple[bytes, int]:
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    backend._check(_fns().acs_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "acs_ipc_export")
    return h.raw, off.value


def ipc_import(handle: bytes, offset: int) -> int:
    p = ctypes.c_void_p()
    backend._check(_fns().acs_ipc_import(handle, offset, ctypes.byref(p)), "acs_ipc_import")
    return p.value


class SlabRank:
    """One rank's slab of a nest: local buffers, neighbour pointers, step loop.

    Neighbour buffers are either raw device pointers of another SlabRank in
    the same process (``connect_local``) or CUDA-IPC imports from other
    processes (``export`` / ``connect_ipc``)."""

    def __init__(self, kernel_id: str, size, nranks: int, rank: int, dtype: str = "f64",
                 variant: str = "accsat", schedule="default"):
        import torch
        self.torch = torch
        self.k = backend.Kernel.lookup(kernel_id)
        self.gw = nests.workload(kernel_id, size, dtype=dtype)
        self.plan = plan_for(self.gw, nranks)
        self.rank, self.nranks = rank, nranks
        self.w = local_workload(self.gw, self.plan, rank)
        self.variant, self.schedule = variant, schedule
        self.nest = self.gw.spec.nest
        self.sharded = [g for grp in ROTATIONS[self.nest] for g in grp]
        self.step_no = 0
        self.buf = self._alloc()
        self.flags = torch.zeros(2, dtype=torch.int64, device="cuda")   # [from lower, from upper]
        self.lo_ptr: Dict[str, int] = {}
        self.hi_ptr: Dict[str, int] = {}
        self.lo_flag = self.hi_flag = None    # neighbours' flag words we signal into
        self.lo_origin = self.hi_origin = 0
        self.imported: List[Tuple[int, int]] = []

    def _alloc(self):
        """Local buffers, filled with the GLOBAL workload's values (flat offset
        of the slab's first plane in the reference layout)."""
        torch = self.torch
        out = {}
        origin = self.plan.origin(self.rank)
        tdt = torch.float32 if self.w.dtype == "f32" else torch.float64
        # every rank allocates the SAME number of planes (the largest slab), so
        # element strides are identical across ranks — the kernel forwards a
        # store to a neighbour at (its own index + a constant plane offset),
        # which must hold for the q-major D3Q19 layout too
        maxp = max(self.plan.local_planes(r) for r in range(self.nranks))
        for p in self.w.spec.arrays:
            dims = self.w.dims[p.name]
            dt = torch.int32 if p.ctype == "int" else tdt
            if len(dims) >= 2:
                full = backend.empty_native(self.k, p.name, (maxp,) + tuple(dims[1:]), dt)
                t = full[:dims[0]]
            else:
                t = backend.empty_native(self.k, p.name, dims, dt)
            out[p.name] = t
        self.refill(out)
        return out

    def refill(self, bufs=None) -> None:
        """(Re)writes the slab's initial values: the GLOBAL workload's stream at
        the slab's reference flat offset, so slabs reproduce the global array."""
        bufs = self.buf if bufs is None else bufs
        origin = self.plan.origin(self.rank)
        for p in self.w.spec.arrays:
            t = bufs[p.name]
            dims = self.w.dims[p.name]
            plane = int(np.prod(dims[1:])) if len(dims) > 1 else 0
            fl = self.w.fills[p.name]
            off = origin * plane if len(dims) > 1 else 0
            if fl.kind == "copy":
                backend.copy(t, bufs[fl.src])
            else:
                lo = fl.value if fl.kind == "const" else fl.lo
                backend.fill(t, fl.kind, nests.SEED_BASE + p.position, lo, fl.hi, fl.p, flat_offset=off)
        self.step_no = 0

    # -- wiring
    def pointers(self) -> Dict[str, int]:
        return {n: t.data_ptr() for n, t in self.buf.items()}

    def connect_local(self, lower: Optional["SlabRank"], upper: Optional["SlabRank"]) -> None:
        if lower is not None:
            self.lo_ptr = {n: lower.buf[n].data_ptr() for n in self.sharded}
            self.lo_origin = lower.plan.origin(lower.rank)
            self.lo_flag = lower.flags.data_ptr() + 8        # lower's "from upper" word
        if upper is not None:
            self.hi_ptr = {n: upper.buf[n].data_ptr() for n in self.sharded}
            self.hi_origin = upper.plan.origin(upper.rank)
            self.hi_flag = upper.flags.data_ptr()            # upper's "from lower" word

    def export(self) -> Dict:
        return {"origin": self.plan.origin(self.rank),
                "bufs": {n: ipc_export(self.buf[n]) for n in self.sharded},
                "flags": ipc_export(self.flags)}

    def connect_ipc(self, lower: Optional[Dict], upper: Optional[Dict]) -> None:
        def imp(h):
            p = ipc_import(*h)
            self.imported.append((p, h[1]))
            return p
        if lower is not None:
            self.lo_ptr = {n: imp(h) for n, h in lower["bufs"].items()}
            self.lo_origin = lower["origin"]
            self.lo_flag = imp(lower["flags"]) + 8
        if upper is not None:
            self.hi_ptr = {n: imp(h) for n, h in upper["bufs"].items()}
            self.hi_origin = upper["origin"]
            self.hi_flag = imp(upper["flags"])

    def close(self) -> None:
        for p, off in self.imported:
            _fns().acs_ipc_close(p, off)
        self.imported = []

    # -- stepping
    def step(self, stream=None, timeout_ms: int = 20000) -> None:
        """One step: wait for the neighbours' previous step, compute the owned
        planes with write-through, signal the neighbours."""
        L = _fns()
        h = backend._stream_handle(stream)
        s = self.step_no
        if s > 0:
            backend._check(L.acs_wait(self.flags.data_ptr() if self.lo_ptr else None,
                                      self.flags.data_ptr() + 8 if self.hi_ptr else None, s, timeout_ms, h),
                           "acs_wait")
        roles = role_buffers(self.nest, [a.name for a in self.w.spec.arrays], s)
        arrays = {p: self.buf[b] for p, b in roles.items()}
        descs, sc = self.k._pack(arrays, dict(self.w.scalars))
        sd = AcsShard()
        lo, hi = self.plan.owned(self.rank)
        sd.own_lo, sd.own_hi, sd.origin, sd.halo = lo, hi, self.plan.origin(self.rank), self.plan.halo
        names = [n for n in self.sharded if n in self.w.write_arrays]   # produced arrays only
        sd.n_sharded = len(names)
        keep = [n.encode() for n in names]
        for i, n in enumerate(names):
            sd.names[i] = keep[i]
            sd.lo_data[i] = self.lo_ptr.get(roles[n]) if self.lo_ptr else None
            sd.hi_data[i] = self.hi_ptr.get(roles[n]) if self.hi_ptr else None
        sd.lo_origin, sd.hi_origin = self.lo_origin, self.hi_origin
        sched = 16 + self.schedule if isinstance(self.schedule, int) else backend.SCHEDULES[self.schedule]
        backend._check(L.acs_launch_sharded(self.k.handle, backend.VARIANTS[self.variant], sched, descs, len(arrays),
                                            sc, len(self.w.scalars), ctypes.byref(sd), h),
                       f"acs_launch_sharded({self.k.kernel_id})")
        if self.lo_flag or self.hi_flag:
            backend._check(L.acs_signal(self.lo_flag, self.hi_flag, s + 1, h), "acs_signal")
        self.step_no = s + 1

    def current(self, name: str):
        """Physical buffer holding parameter `name` after the steps so far."""
        return self.buf[role_buffers(self.nest, [a.name for a in self.w.spec.arrays], self.step_no)[name]]

    def owned_slice(self, name: str):
        """This rank's owned planes of parameter `name` (device tensor view)."""
        lo, hi = self.plan.local_range(self.rank)
        return self.current(name)[lo:hi]
