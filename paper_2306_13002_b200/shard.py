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
ROTATIONS = nests.ROTATIONS
role_buffers = nests.role_buffers


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
    # halo: rows within `halo` of a slab face are written through to the
    # neighbour (never below the upper neighbour's first buffer row); it must
    # not exceed reach_hi (the lower neighbour's window ends reach_hi rows above
    # its owned range)
    halo = {"jacobi7": 1, "wave4": 2, "d3q19": 0, "swim": 1, "clover": 1}[w.spec.nest]
    assert halo <= reach_hi, (w.spec.kernel_id, halo, reach_hi)
    # neighbours exchange only with ranks +-1: every slab must own at least
    # the planes the next step reads across its face (and one plane at all)
    need = max(1, halo, reach_lo, reach_hi)
    if (ghi - glo) // nranks < need:
        raise ValueError(f"{w.spec.kernel_id}: {ghi - glo} planes over {nranks} ranks leaves slabs thinner than "
                         f"the {need} planes a neighbour exchange reaches")
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
        L.acs_signal_ctr.restype = ctypes.c_int
        L.acs_signal_ctr.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.acs_wait_ctr.restype = ctypes.c_int
        L.acs_wait_ctr.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.acs_preload.restype = ctypes.c_int
        L.acs_preload.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(backend.AcsArray), ctypes.c_int,
                                  ctypes.POINTER(backend.AcsScalar), ctypes.c_int]
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


# ---------------------------------------------------------------------------
# message-passing halo exchange (NCCL over NVLink on GPUs, gloo on CPU tensors)

def plane_view(t, lo: int, hi: int):
    """Flat view of planes [lo, hi) of `t` (outermost index) covering exactly
    the elements between the first element of plane lo and the last element
    of plane hi-1 — padded pitches included, so two buffers with the same
    strides exchange the same bytes.  Contiguous, as P2P sends need."""
    torch = backend._torch() if t.is_cuda else __import__("torch")
    if hi <= lo:
        return t.new_empty(0)
    st = t.stride()
    one = 1 + sum((d - 1) * s for d, s in zip(t.shape[1:], st[1:]))
    n = (hi - lo - 1) * st[0] + one
    return torch.as_strided(t, (n,), (1,), t.storage_offset() + lo * st[0])


def written_rows(own: Tuple[int, int], st_lo: int, st_hi: int) -> Tuple[int, int]:
    """Global rows [lo, hi) a rank owning outer-loop range `own` writes into an
    array whose stores reach subscript-0 offsets [st_lo, st_hi]."""
    return own[0] + st_lo, own[1] + st_hi


def exchange_rows(plan: SlabPlan, rank: int, st_lo: int, st_hi: int):
    """Row exchange of one produced array after a kernel, in GLOBAL rows:
    (peer, send rows, recv rows).  A rank sends every row it wrote that lies in
    the neighbour's buffer window and receives every row the neighbour wrote
    that lies in its own — owner computes writes each element exactly once,
    so with row-disjoint stores (store reach of one row) nothing received
    overwrites a row the receiver wrote itself."""
    out = []
    me = written_rows(plan.owned(rank), st_lo, st_hi)
    win = lambda r: (plan.origin(r), plan.origin(r) + plan.local_planes(r))   # noqa: E731
    for peer in (rank - 1, rank + 1):
        if peer < 0 or peer >= plan.nranks:
            continue
        theirs = written_rows(plan.owned(peer), st_lo, st_hi)
        pw, mw = win(peer), win(rank)
        send = (max(me[0], pw[0]), min(me[1], pw[1]))
        recv = (max(theirs[0], mw[0]), min(theirs[1], mw[1]))
        out.append((peer, send, recv))
    return out


def exchange_ops(rank: int, nranks: int, lo: int, hi: int, halo: int):
    """The halo exchange of a produced array whose stores stay on the point's
    own plane, in LOCAL plane coordinates of a rank owning [lo, hi) with a
    `halo`-plane read halo: (peer, send planes, recv planes)."""
    out = []
    if halo <= 0:
        return out
    if rank > 0:
        out.append((rank - 1, (lo, lo + halo), (lo - halo, lo)))
    if rank < nranks - 1:
        out.append((rank + 1, (hi - halo, hi), (hi, hi + halo)))
    return out


def p2p_exchange(dist, t, ops, group=None) -> None:
    """Posts (peer, (send lo, hi), (recv lo, hi)) plane exchanges of `t` as one
    batch of torch.distributed P2P ops (one NCCL group on GPUs) on the CURRENT
    stream and orders later work on that stream after the receives."""
    p2p = []
    for peer, (slo, shi), (rlo, rhi) in ops:
        if shi > slo:
            p2p.append(dist.P2POp(dist.isend, plane_view(t, slo, shi), peer, group))
        if rhi > rlo:
            p2p.append(dist.P2POp(dist.irecv, plane_view(t, rlo, rhi), peer, group))
    if p2p:
        for w in dist.batch_isend_irecv(p2p):
            w.wait()


def halo_exchange(dist, rank: int, nranks: int, t, lo: int, hi: int, halo: int, group=None) -> None:
    """Sends / receives the boundary planes of `t` with ranks +-1 (exchange_ops)."""
    p2p_exchange(dist, t, exchange_ops(rank, nranks, lo, hi, halo), group)


# multi-kernel steps: a benchmark time step of the 2-D nests is a sequence of
# registered regions over the same arrays (SPEC swim: calc1 -> calc2 -> calc3,
# the last copying the new fields back; CloverLeaf: ideal_gas -> PdV ->
# advec_cell x), every kernel over the rank's owned rows
PIPELINES = {
    "swim": ["swim.c:calc1:0", "swim.c:calc2:1", "swim.c:calc3:2"],
    "clover": ["clover.c:ideal_gas:0", "clover.c:pdv_predict:1", "clover.c:advec_cell_x:2"],
}


class SlabRank:
    """One rank's slab of a nest (or of a multi-kernel step): local buffers,
    neighbour pointers, step loop.

    `kernel_id` is one registered region (its time loop rotates buffers per
    nests.ROTATIONS) or a list of regions run in order as one step over the
    union of their arrays (PIPELINES).  Two data paths for the neighbour
    exchange after every kernel:

    * **peer memory** (``connect_local`` / ``connect_ipc``): neighbour buffers
      are raw device pointers (same process, or CUDA-IPC imports over
      NVLink); the compute kernel writes boundary stores through to them and
      device flags order the kernels (``acs_wait_ctr`` / ``acs_signal_ctr``).
      A step is (wait, launch, signal) per kernel with the step count in a
      device counter, so it is captured once per rotation phase as a CUDA
      graph (``capture``) and replayed: no host work per step.
    * **message passing** (``connect_p2p``, NCCL over NVLink when peer
      mapping is unavailable): single-kernel halo nests compute their boundary
      planes first and exchange them on a communication stream while the
      interior planes compute; multi-kernel steps exchange each kernel's
      written rows (``exchange_rows``) before the next kernel.  Row-disjoint
      stores only: D3Q19's push stream writes into rows its neighbours also
      write and needs peer memory."""

    def __init__(self, kernel_id, size, nranks: int, rank: int, dtype: str = "f64",
                 variant: str = "accsat", schedule="default"):
        import torch
        self.torch = torch
        self.ids = [kernel_id] if isinstance(kernel_id, str) else list(kernel_id)
        self.ks = [backend.Kernel.lookup(k) for k in self.ids]
        self.gws = [nests.workload(k, size, dtype=dtype) for k in self.ids]
        self.k, self.gw = self.ks[0], self.gws[0]
        self.plan = plan_for(self.gw, nranks)
        self.rank, self.nranks = rank, nranks
        self.ws = [local_workload(g, self.plan, rank) for g in self.gws]
        self.w = self.ws[0]
        self.variant = variant
        self.schedule = schedule                      # one value, or one per kernel
        self.nest = self.gw.spec.nest
        self.multi = len(self.ids) > 1
        # union of the kernels' arrays (first appearance wins for dims and fill)
        self.arrays: Dict[str, Tuple[nests.ParamSpec, nests.Workload]] = {}
        for lw in self.ws:
            for p in lw.spec.arrays:
                self.arrays.setdefault(p.name, (p, lw))
        self.names = list(self.arrays)
        written = [n for lw in self.ws for n in lw.write_arrays]
        self.sharded = (list(dict.fromkeys(written)) if self.multi
                        else [g for grp in ROTATIONS[self.nest] for g in grp])
        self.period = 1 if self.multi else nests.rotation_period(self.nest)
        self.step_no = 0
        self.buf = self._alloc()
        # [from lower, from upper] step flags (neighbours store into them), and
        # this rank's completed-kernel counter
        self.flags = torch.zeros(2, dtype=torch.int64, device="cuda")
        self.ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.lo_ptr: Dict[str, int] = {}
        self.hi_ptr: Dict[str, int] = {}
        self.lo_flag = self.hi_flag = None    # neighbours' flag words we signal into
        self.lo_origin = self.hi_origin = 0
        self.imported: List[Tuple[int, int]] = []
        self.mode = "none"                    # none | peer | p2p
        self.dist = self.group = None
        self.comm_stream = None
        self.comm_done = None
        self.graphs = None
        self._reach = None
        self.preload()

    def preload(self) -> None:
        """acs_preload for every kernel of the step (see include/accsat_b200.h):
        no kernel code may load lazily while a neighbour's wait kernel spins."""
        L = _fns()
        for ki, (k, lw) in enumerate(zip(self.ks, self.ws)):
            names = [a.name for a in lw.spec.arrays]
            descs, sc = k._pack({n: self.buf[n] for n in names}, dict(lw.scalars))
            backend._check(L.acs_preload(k.handle, backend.VARIANTS[self.variant], descs, len(names), sc,
                                         len(lw.scalars)), f"acs_preload({k.kernel_id})")

    @property
    def points(self) -> int:
        return self.w.points

    @property
    def algorithmic_bytes(self) -> int:
        """This rank's bytes per step (every kernel of the step)."""
        return sum(lw.algorithmic_bytes for lw in self.ws)

    @property
    def global_bytes(self) -> int:
        return sum(g.algorithmic_bytes for g in self.gws)

    def _alloc(self):
        """Local buffers, filled with the GLOBAL workload's values (flat offset
        of the slab's first plane in the reference layout)."""
        torch = self.torch
        out = {}
        tdt = torch.float32 if self.w.dtype == "f32" else torch.float64
        # every rank allocates the SAME number of planes (the largest slab), so
        # element strides are identical across ranks — the kernel forwards a
        # store to a neighbour at (its own index + a constant plane offset),
        # which must hold for the q-major D3Q19 layout too
        maxp = max(self.plan.local_planes(r) for r in range(self.nranks))
        for name, (p, lw) in self.arrays.items():
            dims = lw.dims[name]
            dt = torch.int32 if p.ctype == "int" else tdt
            users = [kk for kk, w in zip(self.ks, self.ws) if name in [a.name for a in w.spec.arrays]]
            k, others = users[0], users[1:]
            if len(dims) >= 2:
                full = backend.empty_native(k, name, (maxp,) + tuple(dims[1:]), dt, shared_with=others)
                t = full[:dims[0]]
            else:
                t = backend.empty_native(k, name, dims, dt, shared_with=others)
            out[name] = t
        self.refill(out)
        return out

    def refill(self, bufs=None) -> None:
        """(Re)writes the slab's initial values: the GLOBAL workload's stream at
        the slab's reference flat offset, so slabs reproduce the global array.
        Also restarts the step count (device counter and flags): call it on
        every rank while no neighbour is stepping, and barrier before the next
        step."""
        bufs = self.buf if bufs is None else bufs
        origin = self.plan.origin(self.rank)
        for name, (p, lw) in self.arrays.items():
            t = bufs[name]
            dims = lw.dims[name]
            plane = int(np.prod(dims[1:])) if len(dims) > 1 else 0
            fl = lw.fills[name]
            off = origin * plane if len(dims) > 1 else 0
            if fl.kind == "copy":
                backend.copy(t, bufs[fl.src])
            else:
                lo = fl.value if fl.kind == "const" else fl.lo
                backend.fill(t, fl.kind, nests.SEED_BASE + p.position, lo, fl.hi, fl.p, flat_offset=off)
        self.step_no = 0
        if hasattr(self, "ctr"):
            self.torch.cuda.synchronize()
            self.flags.zero_()
            self.ctr.zero_()
            self.torch.cuda.synchronize()

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
        self.mode = "peer" if (lower is not None or upper is not None) else "none"
        self.graphs = None

    def export(self) -> Dict:
        return {"origin": self.plan.origin(self.rank),
                "bufs": {n: ipc_export(self.buf[n]) for n in self.sharded},
                "flags": ipc_export(self.flags)}

    def connect_ipc(self, lower: Optional[Dict], upper: Optional[Dict]) -> None:
        def imp(h):
            p = ipc_import(*h)
            self.imported.append((p, h[1]))
            return p
        try:
            if lower is not None:
                self.lo_ptr = {n: imp(h) for n, h in lower["bufs"].items()}
                self.lo_origin = lower["origin"]
                self.lo_flag = imp(lower["flags"]) + 8
            if upper is not None:
                self.hi_ptr = {n: imp(h) for n, h in upper["bufs"].items()}
                self.hi_origin = upper["origin"]
                self.hi_flag = imp(upper["flags"])
        except Exception:
            self.close()
            self.lo_ptr, self.hi_ptr, self.lo_flag, self.hi_flag = {}, {}, None, None
            raise
        self.mode = "peer" if (lower is not None or upper is not None) else "none"
        self.graphs = None

    def reach(self, ki: int) -> Dict[str, "object"]:
        if self._reach is None:
            from . import pipeline_exec
            self._reach = [pipeline_exec.reaches(k) for k in self.ks]
        return self._reach[ki]

    def connect_p2p(self, dist, group=None) -> None:
        """Message-passing exchange through torch.distributed (NCCL)."""
        for ki, lw in enumerate(self.ws):
            for n in lw.write_arrays:
                r = self.reach(ki)[n]
                if r.sliced and r.st_hi != r.st_lo:
                    raise NotImplementedError(
                        f"{self.ids[ki]}: stores of '{n}' reach rows {r.st_lo}..{r.st_hi} around the point — rows "
                        "its neighbours write too (push stream); it needs peer memory (connect_ipc)")
        if not self.multi and self.plan.halo <= 0:
            raise NotImplementedError(f"{self.k.kernel_id}: no halo to exchange; it needs peer memory")
        self.mode = "p2p" if self.nranks > 1 else "none"
        self.dist, self.group = dist, group
        self.comm_stream = self.torch.cuda.Stream()
        self.comm_done = self.torch.cuda.Event()
        self.comm_done.record(self.comm_stream)
        self.graphs = None

    def close(self) -> None:
        for p, off in self.imported:
            _fns().acs_ipc_close(p, off)
        self.imported = []
        self.graphs = None

    # -- stepping
    def _sched(self, ki: int = 0):
        sc = self.schedule[ki] if isinstance(self.schedule, (list, tuple)) else self.schedule
        return 16 + sc if isinstance(sc, int) else backend.SCHEDULES[sc]

    def _launch(self, s: int, h, scalars=None, write_through: bool = True, ki: int = 0) -> None:
        L = _fns()
        lw, k = self.ws[ki], self.ks[ki]
        names = [a.name for a in lw.spec.arrays]
        roles = role_buffers(self.nest, names, s) if not self.multi else {n: n for n in names}
        arrays = {p: self.buf[b] for p, b in roles.items()}
        sc_in = dict(scalars or lw.scalars)
        descs, sc = k._pack(arrays, sc_in)
        sd = AcsShard()
        lo, hi = self.plan.owned(self.rank)
        sd.own_lo, sd.own_hi, sd.origin, sd.halo = lo, hi, self.plan.origin(self.rank), self.plan.halo
        names_wt = [n for n in self.sharded if n in lw.write_arrays] if write_through else []   # produced arrays
        sd.n_sharded = len(names_wt)
        keep = [n.encode() for n in names_wt]
        for i, n in enumerate(names_wt):
            sd.names[i] = keep[i]
            sd.lo_data[i] = self.lo_ptr.get(roles[n]) if self.lo_ptr else None
            sd.hi_data[i] = self.hi_ptr.get(roles[n]) if self.hi_ptr else None
        sd.lo_origin, sd.hi_origin = self.lo_origin, self.hi_origin
        backend._check(L.acs_launch_sharded(k.handle, backend.VARIANTS[self.variant], self._sched(ki), descs,
                                            len(arrays), sc, len(sc_in), ctypes.byref(sd), h),
                       f"acs_launch_sharded({k.kernel_id})")

    def _enqueue_peer(self, s: int, h, timeout_ms: int, before_launch=None) -> None:
        L = _fns()
        neighbours = bool(self.lo_ptr or self.hi_ptr)
        for ki in range(len(self.ks)):
            if neighbours:
                backend._check(L.acs_wait_ctr(self.flags.data_ptr() if self.lo_ptr else None,
                                              self.flags.data_ptr() + 8 if self.hi_ptr else None,
                                              self.ctr.data_ptr(), timeout_ms, h), "acs_wait_ctr")
            if before_launch is not None and ki == 0:
                before_launch(s, h)
            self._launch(s, h, ki=ki)
            if neighbours:
                backend._check(L.acs_signal_ctr(self.lo_flag, self.hi_flag, self.ctr.data_ptr(), h),
                               "acs_signal_ctr")

    def _step_p2p_multi(self, s: int, stream, before_launch=None) -> None:
        """Every kernel over the owned rows, then its written rows exchanged
        with the neighbours before the next kernel."""
        torch = self.torch
        stream = stream or torch.cuda.current_stream()
        h = backend._stream_handle(stream)
        if before_launch is not None:
            before_launch(s, h)
        for ki, lw in enumerate(self.ws):
            self._launch(s, h, write_through=False, ki=ki)
            with torch.cuda.stream(stream):
                for n in lw.write_arrays:
                    r = self.reach(ki)[n]
                    if not r.sliced:
                        continue
                    o = self.plan.origin(self.rank)
                    ops = [(peer, (a - o, b - o), (c - o, d - o))
                           for peer, (a, b), (c, d) in exchange_rows(self.plan, self.rank, r.st_lo, r.st_hi)]
                    p2p_exchange(self.dist, self.buf[n], ops, self.group)

    def _step_p2p(self, s: int, stream, before_launch=None) -> None:
        """Boundary planes, then their exchange on the comm stream overlapped
        with the interior planes."""
        torch = self.torch
        stream = stream or torch.cuda.current_stream()
        h = backend._stream_handle(stream)
        beg, end = self.w.spec.range_params
        lo, hi = self.plan.local_range(self.rank)
        halo = self.plan.halo
        stream.wait_event(self.comm_done)               # halos of the previous step are in place
        if before_launch is not None:
            before_launch(s, h)
        has_lo, has_hi = self.rank > 0, self.rank < self.nranks - 1
        blo = lo + halo if has_lo else lo               # interior [blo, bhi)
        bhi = hi - halo if has_hi else hi
        sc = dict(self.w.scalars)
        for a, b in ((lo, blo), (bhi, hi)):
            if b > a:
                sc[beg], sc[end] = a, b
                self._launch(s, h, sc, write_through=False)
        ev = torch.cuda.Event()
        ev.record(stream)
        out = role_buffers(self.nest, self.names, s)[self.w.write_arrays[0]]
        with torch.cuda.stream(self.comm_stream):
            self.comm_stream.wait_event(ev)
            halo_exchange(self.dist, self.rank, self.nranks, self.buf[out], lo, hi, halo, self.group)
            self.comm_done.record(self.comm_stream)
        if bhi > blo:
            sc[beg], sc[end] = blo, bhi
            self._launch(s, h, sc, write_through=False)

    def step(self, stream=None, timeout_ms: int = 20000, before_launch=None) -> None:
        """One step: wait for the neighbours' previous step, compute the owned
        planes with the exchange, signal the neighbours.  `before_launch(s,
        stream_handle)` (eager steps only) enqueues work that must follow the
        wait and precede the launch, e.g. host uploads into this rank's
        buffers."""
        s = self.step_no
        if self.mode == "p2p":
            if self.multi:
                self._step_p2p_multi(s, stream, before_launch)
            else:
                self._step_p2p(s, stream, before_launch)
        elif self.graphs is not None and before_launch is None:
            with self.torch.cuda.stream(stream or self.torch.cuda.current_stream()):
                self.graphs[s % self.period].replay()
        else:
            self._enqueue_peer(s, backend._stream_handle(stream), timeout_ms, before_launch)
        self.step_no = s + 1

    def capture(self, stream=None, timeout_ms: int = 20000) -> None:
        """Captures one CUDA graph per rotation phase of the peer-memory step
        (per kernel: wait_ctr, launch with write-through, signal_ctr); ``step``
        then replays them.  The device counter carries the step number."""
        if self.mode == "p2p":
            raise RuntimeError("capture: the message-passing step is not captured (NCCL P2P owns its streams)")
        torch = self.torch
        stream = stream or torch.cuda.current_stream()
        cs = torch.cuda.Stream()
        graphs = []
        torch.cuda.synchronize()
        for phase in range(self.period):
            g = torch.cuda.CUDAGraph()
            cs.wait_stream(stream)
            with torch.cuda.graph(g, stream=cs):
                self._enqueue_peer(phase, backend._stream_handle(cs), timeout_ms)
            graphs.append(g)
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        self.graphs = graphs

    def launches_per_step(self) -> int:
        """Kernels this rank enqueues per step (the bench's gpu_launches)."""
        nk = len(self.ks)
        if self.mode == "peer":
            return 3 * nk
        if self.mode == "p2p" and not self.multi:
            return 1 + (self.rank > 0) + (self.rank < self.nranks - 1)
        return nk

    def current(self, name: str):
        """Physical buffer holding parameter `name` after the steps so far."""
        if self.multi:
            return self.buf[name]
        return self.buf[role_buffers(self.nest, self.names, self.step_no)[name]]

    def owned_slice(self, name: str):
        """This rank's owned planes of parameter `name` (device tensor view)."""
        lo, hi = self.plan.local_range(self.rank)
        return self.current(name)[lo:hi]
