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


@pytest.mark.parametrize("kid,size,dtype,nranks", [("wave4.c:wave4:0", (16, 12, 70), "f32", 2),
                                                  ("jacobi7.c:jacobi7:0", (18, 9, 37), "f64", 3),
                                                  ("d3q19.c:stream_collide:0", (12, 7, 20), "f64", 2)])
def test_sharded_graph_capture(kid, size, dtype, nranks):
    """The peer-memory step (wait_ctr, write-through launch, signal_ctr)
    captured once per rotation phase and replayed: bit-exact vs the single
    domain; and N = 1 (no neighbours) is exactly one launch per step."""
    torch = _torch()
    steps = 7
    w, want = single_domain(kid, size, dtype, steps)
    ranks = [shard.SlabRank(kid, size, nranks, r, dtype=dtype, schedule="tiled") for r in range(nranks)]
    for r, sr in enumerate(ranks):
        sr.connect_local(ranks[r - 1] if r > 0 else None, ranks[r + 1] if r < nranks - 1 else None)
    streams = [torch.cuda.Stream() for _ in ranks]
    for sr, st in zip(ranks, streams):
        sr.capture(st)
    for _ in range(steps):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    torch.cuda.synchronize()
    plan = ranks[0].plan
    got = np.concatenate([to_host(sr.owned_slice(LATEST[w.spec.nest])) for sr in ranks], axis=0)
    ref = want[plan.glo:plan.ghi]
    u = np.uint64 if ref.itemsize == 8 else np.uint32
    assert np.array_equal(got.view(u), ref.view(u)), f"{kid} x{nranks}: graph-replayed steps != single domain"
    assert all(int(sr.ctr.item()) == steps for sr in ranks)
    # refill restarts the counters: the same run again from step 0
    for sr in ranks:
        sr.refill()
    for _ in range(steps):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    torch.cuda.synchronize()
    got2 = np.concatenate([to_host(sr.owned_slice(LATEST[w.spec.nest])) for sr in ranks], axis=0)
    assert np.array_equal(got2.view(u), ref.view(u))


def test_one_slab_is_a_plain_launch():
    torch = _torch()
    kid, size = "wave4.c:wave4:0", (10, 9, 40)
    w, want = single_domain(kid, size, "f32", 4)
    sr = shard.SlabRank(kid, size, 1, 0, dtype="f32", schedule="tiled")
    sr.capture()
    for _ in range(4):
        sr.step()
    torch.cuda.synchronize()
    assert sr.mode == "none" and int(sr.ctr.item()) == 0      # no wait / signal kernels
    got = to_host(sr.owned_slice("u"))
    assert np.array_equal(got.view(np.uint32), want[2:12].view(np.uint32))


class _ThreadP2P:
    """In-process stand-in for torch.distributed's P2P API between threads
    (each thread one rank): batch_isend_irecv deposits the sends, meets the
    peer at a barrier and copies the matching receives — so the message-passing
    step (SlabRank.connect_p2p: boundary planes, comm stream, interior planes)
    runs on the device without a second GPU for NCCL."""

    def __init__(self, nranks):
        import threading
        self.bar = threading.Barrier(nranks)
        self.box = {}

    class P2POp:
        def __init__(self, op, tensor, peer, group=None):
            self.op, self.tensor, self.peer = op, tensor, peer

    def isend(self):
        pass

    def irecv(self):
        pass

    def bind(self, rank):
        outer = self

        class View:
            P2POp = _ThreadP2P.P2POp
            isend, irecv = outer.isend, outer.irecv

            @staticmethod
            def batch_isend_irecv(ops):
                import torch
                torch.cuda.current_stream().synchronize()
                for o in ops:
                    if o.op == outer.isend:
                        outer.box[(rank, o.peer)] = o.tensor.clone()
                torch.cuda.current_stream().synchronize()
                outer.bar.wait()
                for o in ops:
                    if o.op == outer.irecv:
                        o.tensor.copy_(outer.box[(o.peer, rank)])
                torch.cuda.current_stream().synchronize()
                outer.bar.wait()
                return []
        return View


@pytest.mark.parametrize("kid,size,dtype,nranks", [("wave4.c:wave4:0", (16, 12, 70), "f32", 2),
                                                  ("wave4.c:wave4:0", (18, 12, 40), "f64", 3),
                                                  ("jacobi7.c:jacobi7:0", (18, 9, 37), "f64", 3)])
def test_sharded_message_passing_step(kid, size, dtype, nranks):
    """connect_p2p: boundary planes first, their halo exchange on a comm
    stream (halo_exchange, the NCCL path) while the interior planes compute;
    bit-exact vs the single domain."""
    import threading
    torch = _torch()
    steps = 5
    w, want = single_domain(kid, size, dtype, steps)
    shim = _ThreadP2P(nranks)
    ranks = [shard.SlabRank(kid, size, nranks, r, dtype=dtype, schedule="tiled") for r in range(nranks)]
    for r, sr in enumerate(ranks):
        sr.connect_p2p(shim.bind(r))
    torch.cuda.synchronize()
    errs = []

    def run(sr):
        try:
            st = torch.cuda.Stream()
            for _ in range(steps):
                sr.step(stream=st)
            st.synchronize()
            sr.comm_stream.synchronize()
        except Exception as e:   # surfaced below
            errs.append(e)
            shim.bar.abort()
    th = [threading.Thread(target=run, args=(sr,)) for sr in ranks]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    torch.cuda.synchronize()
    plan = ranks[0].plan
    got = np.concatenate([to_host(sr.owned_slice(LATEST[w.spec.nest])) for sr in ranks], axis=0)
    ref = want[plan.glo:plan.ghi]
    u = np.uint64 if ref.itemsize == 8 else np.uint32
    assert np.array_equal(got.view(u), ref.view(u)), f"{kid} x{nranks}: message-passing steps != single domain"


def test_message_passing_rejects_push_stream():
    sr = shard.SlabRank("d3q19.c:stream_collide:0", (8, 5, 6), 2, 0)
    with pytest.raises(NotImplementedError):
        sr.connect_p2p(None)


def single_pipeline(nest, size, steps):
    ids = shard.PIPELINES[nest]
    g, ws = nests.pipeline_inputs(ids, size)
    for _ in range(steps):
        for w in ws:
            oracle_cpu.run(w.spec, {p.name: g[p.name] for p in w.spec.arrays}, w.scalars, "accsat", fma=True)
    return g, ws


@pytest.mark.parametrize("nest,size,nranks,sched", [("swim", (24, 70), 2, "tiled"), ("swim", (27, 37), 3, "naive"),
                                                    ("clover", (22, 70), 2, "tiled"), ("clover", (25, 37), 3, "naive")])
@pytest.mark.parametrize("graph", [False, True])
def test_sharded_pipeline_peer(nest, size, nranks, sched, graph):
    """Multi-kernel steps (swim calc1 -> calc2 -> calc3, CloverLeaf ideal_gas ->
    PdV -> advec) slab-sharded with peer write-through after every kernel,
    eager or graph-replayed: bit-exact vs the single domain."""
    torch = _torch()
    steps = 3
    g, ws = single_pipeline(nest, size, steps)
    ids = shard.PIPELINES[nest]
    ranks = [shard.SlabRank(ids, size, nranks, r, schedule=sched) for r in range(nranks)]
    for r, sr in enumerate(ranks):
        sr.connect_local(ranks[r - 1] if r > 0 else None, ranks[r + 1] if r < nranks - 1 else None)
    streams = [torch.cuda.Stream() for _ in ranks]
    if graph:
        for sr, st in zip(ranks, streams):
            sr.capture(st)
    for _ in range(steps):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    torch.cuda.synchronize()
    plan = ranks[0].plan
    bad = []
    for nm in sorted({n for w in ws for n in w.write_arrays}):
        got = np.concatenate([to_host(sr.owned_slice(nm)) for sr in ranks], axis=0)
        if not np.array_equal(got.view(np.uint64), g[nm][plan.glo:plan.ghi].view(np.uint64)):
            bad.append(nm)
    assert not bad, f"{nest} x{nranks}: {bad} differ from the single domain"


@pytest.mark.parametrize("nest,size,nranks", [("swim", (24, 70), 2), ("swim", (27, 37), 3), ("clover", (22, 70), 3)])
def test_sharded_pipeline_message_passing(nest, size, nranks):
    """The NCCL path of a multi-kernel step (each kernel's written rows
    exchanged before the next kernel), with the in-process thread shim."""
    import threading
    torch = _torch()
    steps = 3
    g, ws = single_pipeline(nest, size, steps)
    ids = shard.PIPELINES[nest]
    shim = _ThreadP2P(nranks)
    ranks = [shard.SlabRank(ids, size, nranks, r, schedule="tiled") for r in range(nranks)]
    for r, sr in enumerate(ranks):
        sr.connect_p2p(shim.bind(r))
    torch.cuda.synchronize()
    errs = []

    def run(sr):
        try:
            st = torch.cuda.Stream()
            for _ in range(steps):
                sr.step(stream=st)
            st.synchronize()
        except Exception as e:   # surfaced below
            errs.append(e)
            shim.bar.abort()
    th = [threading.Thread(target=run, args=(sr,)) for sr in ranks]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    torch.cuda.synchronize()
    plan = ranks[0].plan
    for nm in sorted({n for w in ws for n in w.write_arrays}):
        got = np.concatenate([to_host(sr.owned_slice(nm)) for sr in ranks], axis=0)
        assert np.array_equal(got.view(np.uint64), g[nm][plan.glo:plan.ghi].view(np.uint64)), nm
