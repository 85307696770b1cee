"""Slab decomposition — host logic on CPU.

* SlabPlan partitions the outermost loop exactly and sizes local buffers;
* buffer rotation matches the nests' ping-pong / 3-level schemes;
* world_size 2 and 3 over the gloo backend: each rank runs the CPU oracle on
  its slab and exchanges the produced boundary planes with
  ``shard.halo_exchange`` — the code the device path runs over NCCL when peer
  memory is unavailable — and the gathered result equals the single-domain
  run bit for bit (the peer-memory write-through path is checked on the
  device by tests/test_gpu_shard.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cpu as oracle_cpu
from paper_2306_13002_b200 import nests, shard


@pytest.mark.parametrize("kid,size", [("jacobi7.c:jacobi7:0", (11, 5, 6)), ("wave4.c:wave4:0", (13, 4, 5)),
                                      ("d3q19.c:stream_collide:0", (7, 3, 4))])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
def test_slab_plan_partitions(kid, size, nranks):
    w = nests.workload(kid, size)
    plan = shard.plan_for(w, nranks)
    covered = []
    for r in range(nranks):
        lo, hi = plan.owned(r)
        covered.extend(range(lo, hi))
        llo, lhi = plan.local_range(r)
        assert lhi - llo == hi - lo
        assert llo == plan.reach_lo
        lw = shard.local_workload(w, plan, r)
        first = w.spec.arrays[0].name
        assert lw.dims[first][0] == (hi - lo) + plan.reach_lo + plan.reach_hi
        assert lw.dims[first][1:] == w.dims[first][1:]
    assert covered == list(range(plan.glo, plan.ghi))


def test_rotation():
    assert shard.role_buffers("d3q19", ["src", "dst", "flags"], 1) == {"src": "dst", "dst": "src", "flags": "flags"}
    r = shard.role_buffers("wave4", ["u", "up", "un", "vel2"], 1)
    assert (r["up"], r["u"], r["un"]) == ("u", "un", "up")
    assert shard.role_buffers("wave4", ["u", "up", "un", "vel2"], 3)["u"] == "u"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, nranks, port, kid, size, steps, q):
    """One rank: the CPU oracle on its slab (local loop bounds), then the
    produced array's boundary planes exchanged through shard.halo_exchange —
    the same function the device path runs over NCCL (connect_p2p)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    w = nests.workload(kid, size)
    plan = shard.plan_for(w, nranks)
    lw = shard.local_workload(w, plan, rank)
    g = nests.make_inputs(w)
    o = plan.origin(rank)
    n = plan.local_planes(rank)
    loc = {k: np.ascontiguousarray(v[o:o + n]).copy() for k, v in g.items()}
    lo, hi = plan.owned(rank)
    llo, lhi = plan.local_range(rank)
    names = [a.name for a in w.spec.arrays]
    for s in range(steps):
        roles = shard.role_buffers(w.spec.nest, names, s)
        arrs = {p: loc[b] for p, b in roles.items()}
        oracle_cpu.run(w.spec, arrs, lw.scalars, "accsat", fma=True)
        out = roles[w.write_arrays[0]]
        shard.halo_exchange(dist, rank, nranks, torch.from_numpy(loc[out]), llo, lhi, plan.halo)
    latest = {"jacobi7": "A0", "wave4": "u", "d3q19": "src"}[w.spec.nest]   # holds the newest field
    final = shard.role_buffers(w.spec.nest, names, steps)[latest]
    part = loc[final][lo - o:hi - o]
    parts = [None] * nranks
    dist.all_gather_object(parts, part)
    if rank == 0:
        q.put(np.concatenate(parts, axis=0))
    dist.destroy_process_group()


def test_exchange_ops():
    assert shard.exchange_ops(0, 1, 2, 10, 2) == []
    assert shard.exchange_ops(0, 3, 2, 10, 2) == [(1, (8, 10), (10, 12))]
    assert shard.exchange_ops(1, 3, 2, 10, 2) == [(0, (2, 4), (0, 2)), (2, (8, 10), (10, 12))]
    assert shard.exchange_ops(2, 3, 1, 5, 0) == []


def test_plane_view_covers_padded_planes():
    t = torch.arange(5 * 3 * 8, dtype=torch.float64).reshape(5, 3, 8)[:, :, :6]   # padded pitch
    v = shard.plane_view(t, 1, 3)
    assert v.is_contiguous() and v.numel() == 8 * 3 + 2 * 8 + 6
    assert v[0].item() == t[1, 0, 0].item() and v[-1].item() == t[2, 2, 5].item()


def test_plan_rejects_thin_slabs():
    w = nests.workload("wave4.c:wave4:0", (5, 4, 4))
    with pytest.raises(ValueError):
        shard.plan_for(w, 3)      # 1-plane slabs, halo 2
    shard.plan_for(w, 2)


@pytest.mark.parametrize("kid,size,steps,nranks", [("jacobi7.c:jacobi7:0", (9, 6, 7), 3, 2),
                                                 ("wave4.c:wave4:0", (11, 5, 6), 4, 2),
                                                 ("wave4.c:wave4:0", (13, 5, 6), 5, 3)])
def test_gloo_ranks_equal_single_domain(kid, size, steps, nranks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, nranks, port, kid, size, steps, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single domain
    w = nests.workload(kid, size)
    g = nests.make_inputs(w)
    names = [a.name for a in w.spec.arrays]
    for s in range(steps):
        roles = shard.role_buffers(w.spec.nest, names, s)
        oracle_cpu.run(w.spec, {p: g[b] for p, b in roles.items()}, w.scalars, "accsat", fma=True)
    final = shard.role_buffers(w.spec.nest, names, steps)["A0" if w.spec.nest == "jacobi7" else "u"]
    plan = shard.plan_for(w, nranks)
    want = g[final][plan.glo:plan.ghi]
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_exchange_rows_swim_pattern():
    """swim calc1 writes cv/z at j+1: rank r sends row own_hi to the upper
    neighbour and never row own_hi-1 (outside the upper's buffer)."""
    w = nests.workload("swim.c:calc1:0", (12, 9))
    plan = shard.plan_for(w, 3)             # owned [0,4) [4,8) [8,12), reach (0, 1)
    ops = dict((p, (s, r)) for p, s, r in shard.exchange_rows(plan, 1, 1, 1))
    assert ops[2] == ((8, 9), (9, 9))       # send row 8 up, nothing comes down for a j+1 store
    assert ops[0] == ((5, 5), (4, 5))       # lower's row 4 arrives
    ops0 = dict((p, (s, r)) for p, s, r in shard.exchange_rows(plan, 1, 0, 0))
    assert ops0[0] == ((4, 5), (4, 4)) and ops0[2] == ((8, 8), (8, 9))


def _pipeline_worker(rank, nranks, port, nest, size, steps, q):
    """A multi-kernel step (swim calc1->calc2->calc3, CloverLeaf ideal_gas ->
    PdV -> advec) on one rank's rows: every kernel through the CPU oracle on
    the slab, then its written rows exchanged with shard.p2p_exchange over the
    rows shard.exchange_rows names — the NCCL path of SlabRank.connect_p2p."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    from paper_2306_13002_b200 import backend, pipeline_exec
    ids = shard.PIPELINES[nest]
    g, ws = nests.pipeline_inputs(ids, size)
    plan = shard.plan_for(ws[0], nranks)
    o, n = plan.origin(rank), plan.local_planes(rank)
    loc = {k: np.ascontiguousarray(v[o:o + n]).copy() if v.ndim >= 2 else v.copy() for k, v in g.items()}
    reach = [pipeline_exec.reaches(backend.Kernel.lookup(k)) for k in ids]
    for _ in range(steps):
        for ki, w in enumerate(ws):
            lw = shard.local_workload(w, plan, rank)
            oracle_cpu.run(w.spec, {p.name: loc[p.name] for p in w.spec.arrays}, lw.scalars, "accsat", fma=True)
            for name in w.write_arrays:
                r = reach[ki][name]
                ops = [(peer, (a - o, b - o), (c - o, d - o))
                       for peer, (a, b), (c, d) in shard.exchange_rows(plan, rank, r.st_lo, r.st_hi)]
                shard.p2p_exchange(dist, torch.from_numpy(loc[name]), ops)
    lo, hi = plan.owned(rank)
    written = sorted({nm for w in ws for nm in w.write_arrays})
    part = {nm: loc[nm][lo - o:hi - o] for nm in written}
    parts = [None] * nranks
    dist.all_gather_object(parts, part)
    if rank == 0:
        q.put({nm: np.concatenate([p[nm] for p in parts], axis=0) for nm in written})
    dist.destroy_process_group()


@pytest.mark.parametrize("nest,size,steps,nranks", [("swim", (13, 17), 3, 2), ("swim", (14, 9), 2, 3),
                                                    ("clover", (11, 13), 2, 2)])
def test_gloo_pipeline_equals_single_domain(nest, size, steps, nranks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, nranks, port, nest, size, steps, q))
             for r in range(nranks)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = shard.PIPELINES[nest]
    g, ws = nests.pipeline_inputs(ids, size)
    for _ in range(steps):
        for w in ws:
            oracle_cpu.run(w.spec, {p.name: g[p.name] for p in w.spec.arrays}, w.scalars, "accsat", fma=True)
    plan = shard.plan_for(ws[0], nranks)
    for nm, arr in got.items():
        want = g[nm][plan.glo:plan.ghi]
        assert np.array_equal(arr.view(np.uint64), want.view(np.uint64)), nm
