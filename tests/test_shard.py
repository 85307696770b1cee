"""Slab decomposition — host logic on CPU.

* SlabPlan partitions the outermost loop exactly and sizes local buffers;
* buffer rotation matches the nests' ping-pong / 3-level schemes;
* an emulation of owner-computes + halo write-through with world_size 2 over
  the gloo backend, each rank running the CPU oracle on its slab, reproduces
  the single-domain result bit for bit (the device path does the same
  forwarding from inside the kernel; tests/test_gpu_shard.py checks that)."""
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
    names = [a.name for a in w.spec.arrays]
    for s in range(steps):
        roles = shard.role_buffers(w.spec.nest, names, s)
        arrs = {p: loc[b] for p, b in roles.items()}
        oracle_cpu.run(w.spec, arrs, lw.scalars, "accsat", fma=True)
        # write-through of the produced array's boundary planes (whole planes:
        # the owner rewrites every element of its owned planes each step)
        out = roles[w.write_arrays[0]]
        h = plan.halo
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(loc[out][lo - o:lo - o + h].copy()), rank - 1))
        if rank < nranks - 1:
            reqs.append(dist.isend(torch.from_numpy(loc[out][hi - o - h:hi - o].copy()), rank + 1))
        if rank > 0:
            buf = torch.from_numpy(np.empty_like(loc[out][:h]))
            dist.recv(buf, rank - 1)
            lo_o = plan.origin(rank - 1)
            lo_hi = plan.owned(rank - 1)[1]
            loc[out][lo_hi - h - o:lo_hi - o] = buf.numpy()
        if rank < nranks - 1:
            buf = torch.from_numpy(np.empty_like(loc[out][:h]))
            dist.recv(buf, rank + 1)
            up_lo = plan.owned(rank + 1)[0]
            loc[out][up_lo - o:up_lo + h - o] = buf.numpy()
        for r in reqs:
            r.wait()
    latest = {"jacobi7": "A0", "wave4": "u", "d3q19": "src"}[w.spec.nest]   # holds the newest field
    final = shard.role_buffers(w.spec.nest, names, steps)[latest]
    part = loc[final][lo - o:hi - o]
    parts = [None] * nranks
    dist.all_gather_object(parts, part)
    if rank == 0:
        q.put(np.concatenate(parts, axis=0))
    dist.destroy_process_group()


@pytest.mark.parametrize("kid,size,steps", [("jacobi7.c:jacobi7:0", (9, 6, 7), 3), ("wave4.c:wave4:0", (11, 5, 6), 4)])
def test_gloo_two_ranks_equal_single_domain(kid, size, steps):
    nranks = 2
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
