"""GPU parity at every configured BASELINE size, and on edge-value inputs.

Everything here runs the same code the bench times and compares it, bit for
bit, with the reference's CPU path on the same inputs (the compiled
reference text, OpenMP; oracle/):

* every nest x every form (original, cse, cse+bulk, cse+sat, accsat) at its
  BASELINE grid — wave4 1024^3 fp32 (4.35 GB per field, past 2^32 bytes) and
  zsolve 256^3 included — on the naive skeleton and on the slot the tuner
  picks for that form;
* Jacobi's 100-sweep step as the CUDA graph the bench replays;
* wave4's multi-step 3-level rotation through the slab path (N = 1), the
  bench's headline path, graph-replayed;
* the e2e host-buffer path (HostRunner, 16 chunks) at full size for D3Q19
  256^3 and wave4 1024^3;
* edge values (zeros, subnormals, +-inf, NaN, huge magnitudes, and the
  reference random_env distribution U[-10, 10] / ints U[1, 8],
  proj/src/interp.cpp:272-298) with a NaN-equal comparison: NaN matches NaN
  of any payload (GPU and glibc payloads differ), everything else bitwise.
"""
import os

import numpy as np
import pytest

import cpu as oracle_cpu
from paper_2306_13002_b200 import backend, nests

pytestmark = pytest.mark.gpu

VARIANTS = ["original", "cse", "cse+bulk", "cse+sat", "accsat"]
SAT = {"cse+sat", "accsat"}
THREADS = os.cpu_count() or 1

FULL = [("jacobi7.c:jacobi7:0", 256, "f64"), ("d3q19.c:stream_collide:0", 256, "f64"),
        ("swim.c:calc1:0", 8192, "f64"), ("swim.c:calc2:1", 8192, "f64"), ("swim.c:calc3:2", 8192, "f64"),
        ("clover.c:ideal_gas:0", 7680, "f64"), ("clover.c:pdv_predict:1", 7680, "f64"),
        ("clover.c:advec_cell_x:2", 7680, "f64"), ("wave4.c:wave4:0", 1024, "f32"),
        ("zsolve.c:z_solve_lhs:0", 256, "f64")]


def _torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def to_host(t):
    torch = _torch()
    if not t.is_contiguous():
        rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
        backend.copy(rm, t)
        t = rm
    torch.cuda.synchronize()
    out = t.cpu().numpy()
    del t
    return out


def n_diff(a, b, nan_equal=False):
    """Elements whose bits differ (NaN vs NaN counted equal with nan_equal)."""
    if a.dtype.kind != "f":
        return int(np.count_nonzero(a != b))
    u = np.uint64 if a.itemsize == 8 else np.uint32
    ne = a.view(u) != b.view(u)
    if nan_equal:
        ne &= ~(np.isnan(a) & np.isnan(b))
    return int(np.count_nonzero(ne))


def oracle(w, host, variant, steps=1):
    """The reference's CPU path on copies of the written arrays (read-only
    arrays shared), `steps` steps with the nest's buffer rotation."""
    written = set(w.write_arrays)
    for grp in nests.ROTATIONS.get(w.spec.nest, []):
        written |= set(grp)
    arrs = {n: (a.copy() if n in written else a) for n, a in host.items()}
    names = list(arrs)
    for s in range(steps):
        roles = nests.role_buffers(w.spec.nest, names, s)
        oracle_cpu.run(w.spec, {p: arrs[b] for p, b in roles.items()}, w.scalars, variant, fma=variant in SAT,
                       f32=w.dtype == "f32", threads=THREADS)
    return arrs, nests.role_buffers(w.spec.nest, names, steps)


@pytest.mark.parametrize("kid,size,dtype", FULL, ids=[f[0].split(":")[1] for f in FULL])
def test_full_size_every_form_naive_and_tuned(kid, size, dtype):
    torch = _torch()
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    host = oracle_cpu.host_inputs(w, THREADS)
    prec = 1 if dtype == "f32" else 0
    bad = []
    for variant in VARIANTS:
        want, _ = oracle(w, host, variant)
        dev = nests.device_inputs(w, native=True, kernel=k)
        tuned, _ = k.tune(dev, dict(w.scalars), variant, reps=1)
        del dev
        for slot in sorted({0, tuned}):
            dev = nests.device_inputs(w, native=True, kernel=k)       # fresh inputs
            k.launch(dev, dict(w.scalars), variant, slot)
            for n in w.write_arrays:
                d = n_diff(to_host(dev[n]), want[n])
                if d:
                    bad.append(f"{variant}/slot {slot} ({k.info['schedules'][prec][slot]}): '{n}' {d} elements")
            del dev
            torch.cuda.empty_cache()
        del want
    assert not bad, f"{kid} at {size}: " + "; ".join(bad)


@pytest.mark.parametrize("variant,schedule", [("original", "naive"), ("accsat", "default")])
def test_jacobi_100_sweep_graph_step_full_size(variant, schedule):
    """The bench's Jacobi step: one CUDA graph of 100 ping-pong launches at
    256^3, replayed; after the capture's warm step and two replays (300
    sweeps) A0 equals 300 sweeps of the compiled reference text."""
    torch = _torch()
    from paper_2306_13002_b200 import stepper
    kid = "jacobi7.c:jacobi7:0"
    w = nests.workload(kid, 256)
    k = backend.Kernel.lookup(kid)
    dev = nests.device_inputs(w, native=True, kernel=k)
    if schedule == "default":
        k.tune(dev, dict(w.scalars), variant, reps=1)
        dev = nests.device_inputs(w, native=True, kernel=k)
    st = stepper.Stepper(k, dev, w.scalars, variant, schedule, sweeps=100)
    st.capture()
    st.step()
    st.step()
    assert st.t == 300
    got = to_host(st.current("A0"))
    host = oracle_cpu.host_inputs(w, THREADS)
    want, roles = oracle(w, host, variant, steps=300)
    assert n_diff(got, want[roles["A0"]]) == 0


def test_wave4_slab_path_multi_step_full_size():
    """The headline path: wave4 1024^3 fp32 accsat through SlabRank (one
    slab), tuned, graph-captured, 4 steps (one full 3-level rotation + 1)."""
    torch = _torch()
    from paper_2306_13002_b200 import shard
    kid, steps = "wave4.c:wave4:0", 4
    sr = shard.SlabRank(kid, (1024,) * 3, 1, 0, dtype="f32")
    sr.schedule, _ = sr.k.tune(sr.buf, dict(sr.w.scalars), "accsat", reps=1)
    sr.refill()
    sr.capture()
    for _ in range(steps):
        sr.step()
    torch.cuda.synchronize()
    got = {p: to_host(sr.current(p)) for p in ("u", "up")}
    sr.close()
    del sr
    torch.cuda.empty_cache()
    w = nests.workload(kid, 1024, dtype="f32")
    want, roles = oracle(w, oracle_cpu.host_inputs(w, THREADS), "accsat", steps=steps)
    for p in ("u", "up"):
        assert n_diff(got[p], want[roles[p]]) == 0, p


@pytest.mark.parametrize("kid,size,dtype", [("d3q19.c:stream_collide:0", 256, "f64"),
                                            ("wave4.c:wave4:0", 1024, "f32")])
def test_host_runner_full_size(kid, size, dtype):
    """The bench's e2e path (pinned reference-layout host buffers, 16 chunks,
    graph-captured) at the BASELINE grid, with the device staging poisoned."""
    torch = _torch()
    from paper_2306_13002_b200 import pipeline_exec
    w = nests.workload(kid, size, dtype=dtype)
    k = backend.Kernel.lookup(kid)
    host_np = oracle_cpu.host_inputs(w, THREADS)
    want, _ = oracle(w, host_np, "accsat")
    host = {n: torch.from_numpy(a).pin_memory() for n, a in host_np.items()}
    del host_np
    r = pipeline_exec.HostRunner(k, host, w.spec.range_params, chunks=16)
    for n in host:
        for t in (r.rm[n], r.nat[n]):
            t.fill_(float("nan") if t.dtype.is_floating_point else -12345)
    g = r.capture(dict(w.scalars), "accsat")
    g.replay()                    # capture ran the call once already: same inputs, same result
    torch.cuda.synchronize()
    for n in w.write_arrays:
        assert n_diff(host[n].numpy(), want[n]) == 0, n


# ---- edge values ---------------------------------------------------------------

EDGE_SIZES = {"jacobi7": (6, 7, 19), "wave4": (6, 5, 21), "d3q19": (4, 5, 11), "swim": (9, 23),
              "clover": (9, 23), "zsolve": (3, 4, 9)}


def edge_inputs(w, kind, seed=7):
    """'special': a seeded mix of zeros, +-0, subnormals, +-inf, NaN and huge
    values sprinkled into the workload's inputs; 'random_env': every element
    U[-10, 10] (ints U[1, 8]) like the reference's random_env."""
    rng = np.random.default_rng(seed)
    base = nests.make_inputs(w)
    out = {}
    for n, a in base.items():
        a = a.copy()
        flat = a.reshape(-1)
        if a.dtype.kind != "f":
            if kind == "random_env":
                flat[:] = rng.integers(1, 9, flat.size)
            out[n] = a
            continue
        if kind == "random_env":
            flat[:] = rng.uniform(-10.0, 10.0, flat.size)
        else:
            tiny = np.finfo(a.dtype).tiny
            specials = np.array([0.0, -0.0, tiny / 4, -tiny / 3, tiny, np.inf, -np.inf, np.nan,
                                 np.finfo(a.dtype).max / 8, -1e30 if a.dtype == np.float32 else -1e300],
                                dtype=a.dtype)
            pick = rng.random(flat.size) < 0.2
            flat[pick] = specials[rng.integers(0, specials.size, int(pick.sum()))]
        out[n] = a
    return out


def edge_cases():
    out = []
    for kid, spec in nests.KERNELS.items():
        for dtype in (("f64", "f32") if spec.nest == "wave4" else ("f64",)):
            for kind in ("special", "random_env"):
                out.append((kid, dtype, kind))
    return out


@pytest.mark.parametrize("kid,dtype,kind", edge_cases(),
                         ids=[f"{c[0].split(':')[1]}-{c[1]}-{c[2]}" for c in edge_cases()])
def test_edge_values_nan_equal(kid, dtype, kind):
    """Every form on every registered slot: bitwise equal to the compiled
    reference text on inputs full of special values (NaN-equal)."""
    torch = _torch()
    spec = nests.kernel(kid)
    w = nests.workload(kid, EDGE_SIZES[spec.nest], dtype=dtype)
    ins = edge_inputs(w, kind)
    k = backend.Kernel.lookup(kid)
    prec = 1 if dtype == "f32" else 0
    slots = [i for i, nm in enumerate(k.info["schedules"][prec]) if nm]
    bad = []
    for variant in VARIANTS:
        want = {n: a.copy() for n, a in ins.items()}
        oracle_cpu.run(spec, want, w.scalars, variant, fma=variant in SAT, f32=dtype == "f32")
        for slot in slots:
            dev = {}
            for n, a in ins.items():
                t = torch.from_numpy(a.copy()).cuda()
                d = backend.empty_native(k, n, a.shape, t.dtype)
                backend.copy(d, t)
                dev[n] = d
            k.launch(dev, dict(w.scalars), variant, slot)
            for n in w.write_arrays:
                nd = n_diff(to_host(dev[n]), want[n], nan_equal=True)
                if nd:
                    bad.append(f"{variant}/slot {slot}: '{n}' {nd} elements")
    assert not bad, f"{kid} {dtype} {kind}: " + "; ".join(bad)
