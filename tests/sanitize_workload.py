"""Small launches of every skeleton, run under compute-sanitizer by
tests/test_gpu_sanitizer.py (memcheck / racecheck / synccheck).

Every registered schedule slot of every nest (naive, march TMA ring,
register windows, stream cp.async ring, sliced register queue) in the
original and accsat forms on ragged grids, the wave4 fp32 instantiation, the
host-buffer pipeline, and a 2-slab sharded time loop on one device (peer
write-through stores + device step flags, graph-replayed) — each checked
against the CPU oracle so a silently wrong kernel fails here too.

usage: python tests/sanitize_workload.py [quick]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import cpu as oracle_cpu  # noqa: E402
from paper_2306_13002_b200 import backend, nests, shard  # noqa: E402

SIZES = {"jacobi7": (5, 6, 37), "wave4": (6, 5, 37), "d3q19": (3, 4, 20), "swim": (9, 37), "clover": (9, 37),
         "zsolve": (3, 2, 20)}


def to_host(t):
    import torch
    if not t.is_contiguous():
        rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
        backend.copy(rm, t)
        t = rm
    torch.cuda.synchronize()
    return t.cpu().numpy()


def check(kid, dtype, variants=("original", "accsat")):
    import torch
    spec = nests.kernel(kid)
    w = nests.workload(kid, SIZES[spec.nest], dtype=dtype)
    ins = nests.make_inputs(w)
    k = backend.Kernel.lookup(kid)
    prec = 1 if dtype == "f32" else 0
    for variant in variants:
        want = {n: a.copy() for n, a in ins.items()}
        oracle_cpu.run(spec, want, w.scalars, variant, fma=variant == "accsat", f32=dtype == "f32")
        for slot, name in enumerate(k.info["schedules"][prec]):
            if not name:
                continue
            dev = {}
            for n, a in ins.items():
                t = torch.from_numpy(a.copy()).cuda()
                d = backend.empty_native(k, n, a.shape, t.dtype)
                backend.copy(d, t)
                dev[n] = d
            k.launch(dev, dict(w.scalars), variant, slot)
            for n in w.write_arrays:
                got = to_host(dev[n])
                u = np.uint64 if got.itemsize == 8 else np.uint32
                assert np.array_equal(got.view(u), want[n].view(u)), f"{kid} {variant} slot {slot} ({name})"


def sharded(kid, size, dtype, steps=4):
    import torch
    ranks = [shard.SlabRank(kid, size, 2, r, dtype=dtype, schedule="tiled") for r in range(2)]
    ranks[0].connect_local(None, ranks[1])
    ranks[1].connect_local(ranks[0], None)
    streams = [torch.cuda.Stream() for _ in ranks]
    for sr, st in zip(ranks, streams):
        sr.capture(st)
    for _ in range(steps):
        for sr, st in zip(ranks, streams):
            sr.step(stream=st)
    torch.cuda.synchronize()
    w = nests.workload(kid, size, dtype=dtype)
    g = nests.make_inputs(w)
    names = [a.name for a in w.spec.arrays]
    for s in range(steps):
        roles = nests.role_buffers(w.spec.nest, names, s)
        oracle_cpu.run(w.spec, {p: g[b] for p, b in roles.items()}, w.scalars, "accsat", fma=True,
                       f32=dtype == "f32")
    latest = {"jacobi7": "A0", "wave4": "u", "d3q19": "src"}[w.spec.nest]
    want = g[nests.role_buffers(w.spec.nest, names, steps)[latest]]
    got = np.concatenate([to_host(sr.owned_slice(latest)) for sr in ranks], axis=0)
    plan = ranks[0].plan
    u = np.uint64 if got.itemsize == 8 else np.uint32
    assert np.array_equal(got.view(u), want[plan.glo:plan.ghi].view(u)), f"sharded {kid}"


def host_runner():
    import torch
    from paper_2306_13002_b200 import pipeline_exec
    kid = "d3q19.c:stream_collide:0"
    w = nests.workload(kid, (5, 4, 11))
    ins = nests.make_inputs(w)
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(w.spec, want, w.scalars, "accsat", fma=True)
    host = {n: torch.from_numpy(a.copy()).pin_memory() for n, a in ins.items()}
    r = pipeline_exec.HostRunner(backend.Kernel.lookup(kid), host, w.spec.range_params, chunks=3)
    r.run(dict(w.scalars), "accsat")
    torch.cuda.synchronize()
    assert np.array_equal(host["dst"].numpy().view(np.uint64), want["dst"].view(np.uint64))


def main():
    import torch
    torch.cuda.set_device(0)
    quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
    kids = sorted(nests.KERNELS)
    if quick:
        kids = ["jacobi7.c:jacobi7:0", "wave4.c:wave4:0", "zsolve.c:z_solve_lhs:0", "d3q19.c:stream_collide:0",
                "clover.c:advec_cell_x:2"]
    for kid in kids:
        check(kid, "f64", ("accsat",) if quick else ("original", "accsat"))
    check("wave4.c:wave4:0", "f32", ("accsat",))
    sharded("wave4.c:wave4:0", (12, 6, 37), "f32")
    sharded("jacobi7.c:jacobi7:0", (10, 5, 19), "f64")
    sharded("d3q19.c:stream_collide:0", (8, 4, 11), "f64")
    host_runner()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
