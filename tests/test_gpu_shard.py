"""Slab-sharded execution on the device: owner computes, stores written
through to the neighbours' buffers from inside the kernel, steps ordered by
device-side flags.  Several slabs share one GPU here (the driver's boxes have
one), exactly as separate GPUs would over NVLink: the kernels only see device
pointers.  Parity: the gathered owned planes after T steps equal the
single-domain run bit for bit (and the CPU oracle)."""
import os
import socket

import numpy as np
import pytest

import cpu as oracle_cpu
from paper_2306_13002_b200 import backend, nests, shard

pytestmark = pytest.mark.gpu

LATEST = {"jacobi7": "A0", "wave4": "u", "d3q19": "src"}


def _torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def single_domain(kid, size, dtype, steps):
    """CPU oracle, T steps of the whole domain (fma form = what the GPU computes)."""
    w = nests.workload(kid, size, dtype=dtype)
    g = nests.make_inputs(w)
    names = [a.name for a in w.spec.arrays]
    for s in range(steps):
        roles = shard.role_buffers(w.spec.nest, names, s)
        oracle_cpu.run(w.spec, {p: g[b] for p, b in roles.items()}, w.scalars, "accsat", fma=True,
                       f32=dtype == "f32")
    return w, g[shard.role_buffers(w.spec.nest, names, steps)[LATEST[w.spec.nest]]]


def to_host(t):
    torch = _torch()
    if not t.is_contiguous():
        rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
        backend.copy(rm, t)
        t = rm
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("kid,size,dtype", [
    ("jacobi7.c:jacobi7:0", (12, 9, 37), "f64"),
    ("wave4.c:wave4:0", (13, 10, 35), "f64"),
    ("wave4.c:wave4:0", (16, 12, 70), "f32"),
    ("d3q19.c:stream_collide:0", (9, 7, 20), "f64"),
])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("sched", ["naive", "tiled"])
def test_sharded_equals_single_domain(kid, size, dtype, nranks, sched):
    torch = _torch()
    steps = 4
    w, want = single_domain(kid, size, dtype, steps)
    ranks = [shard.SlabRank(kid, size, nranks, r, dtype=dtype, schedule=sched) for r in range(nranks)]
    for r, sr in enumerate(ranks):
        sr.connect_local(ranks[r - 1] if r > 0 else None, ranks[r + 1] if r < nranks - 1 else None)
    streams = [torch.cuda.Stream() for _ in ranks]
    torch.cuda.synchronize()
    for _ in range(steps):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    torch.cuda.synchronize()
    plan = ranks[0].plan
    got = np.concatenate([to_host(sr.owned_slice(LATEST[w.spec.nest])) for sr in ranks], axis=0)
    ref = want[plan.glo:plan.ghi]
    u = np.uint64 if ref.itemsize == 8 else np.uint32
    assert np.array_equal(got.view(u), ref.view(u)), f"{kid} x{nranks} {sched}: sharded != single domain"


def _slots(kid, prec):
    k = backend.Kernel.lookup(kid)
    return [i for i, n in enumerate(k.info["schedules"][prec]) if n]


@pytest.mark.parametrize("kid,size,dtype,prec", [("wave4.c:wave4:0", (40, 12, 70), "f32", 1),
                                                 ("jacobi7.c:jacobi7:0", (36, 9, 37), "f64", 0),
                                                 ("d3q19.c:stream_collide:0", (24, 7, 20), "f64", 0)])
def test_sharded_every_slot(kid, size, dtype, prec):
    """Every registered schedule slot (register windows with deferred vector
    stores on interior planes included) with 2 slabs thick enough to have
    planes away from the faces: bit-exact vs the single domain."""
    torch = _torch()
    steps = 3
    w, want = single_domain(kid, size, dtype, steps)
    for slot in _slots(kid, prec):
        ranks = [shard.SlabRank(kid, size, 2, r, dtype=dtype, schedule=slot) for r in range(2)]
        ranks[0].connect_local(None, ranks[1])
        ranks[1].connect_local(ranks[0], None)
        streams = [torch.cuda.Stream() for _ in ranks]
        torch.cuda.synchronize()
        for _ in range(steps):
            for sr, st in zip(ranks, streams):
                sr.step(stream=st)
        torch.cuda.synchronize()
        plan = ranks[0].plan
        got = np.concatenate([to_host(sr.owned_slice(LATEST[w.spec.nest])) for sr in ranks], axis=0)
        ref = want[plan.glo:plan.ghi]
        u = np.uint64 if ref.itemsize == 8 else np.uint32
        assert np.array_equal(got.view(u), ref.view(u)), f"{kid} slot {slot}: sharded != single domain"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, nranks, port, kid, size, steps, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    torch.cuda.set_device(0)
    sr = shard.SlabRank(kid, size, nranks, rank)
    torch.cuda.synchronize()
    exp = [None] * nranks
    dist.all_gather_object(exp, sr.export())
    sr.connect_ipc(exp[rank - 1] if rank > 0 else None, exp[rank + 1] if rank < nranks - 1 else None)
    dist.barrier()
    for _ in range(steps):
        sr.step()
    torch.cuda.synchronize()
    dist.barrier()
    part = to_host(sr.owned_slice(LATEST[sr.nest]))
    parts = [None] * nranks
    dist.all_gather_object(parts, part)
    sr.close()
    if rank == 0:
        q.put(np.concatenate(parts, axis=0))
    dist.destroy_process_group()


def test_two_processes_cuda_ipc():
    """Two processes, buffers exchanged with CUDA IPC (the multi-GPU path;
    here both processes share the one GPU)."""
    import torch.multiprocessing as mp
    kid, size, steps, nranks = "wave4.c:wave4:0", (12, 9, 33), 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, nranks, port, kid, size, steps, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w, want = single_domain(kid, size, "f64", steps)
    plan = shard.plan_for(w, nranks)
    assert np.array_equal(got.view(np.uint64), want[plan.glo:plan.ghi].view(np.uint64))
