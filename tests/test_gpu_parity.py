"""GPU parity: every registered nest x variant x skeleton, through the C ABI,
against the CPU oracle on the same seeded inputs.

* ORIGINAL / CSE / CSE_BULK forms: BIT-EXACT against the compiled reference
  text (gcc -ffp-contract=off), which tests/test_oracle.py pins bit-exact to
  the reference interpreter.
* CSE_SAT / ACCSAT forms compute each extracted FMA with ONE rounding on the
  GPU, so they are compared BIT-EXACT against the FMA-rewritten reference text
  (oracle ``*_fma``), and — against the two-rounding reference interpreter
  itself — within the reference comparator's rule |d| <= 1e-12*max(|a|,|b|)
  or |d| <= 1e-12 (proj/src/oracle.cpp:12, :30-38) for fp64.
* wave4 fp32: bit-exact against the fp32 textual copy (fmaf-rewritten for the
  saturated forms); vs the fp64 text within 1e-5 with a norm-wise floor
  1e-5*max|ref|.
"""
import glob
import json
import os

import numpy as np
import pytest

import cpu as oracle_cpu
from paper_2306_13002_b200 import backend, nests

pytestmark = pytest.mark.gpu

VARIANTS = ["original", "cse", "cse+bulk", "cse+sat", "accsat"]
SAT = {"cse+sat", "accsat"}

# (kernel nest, sizes) — ragged and odd extents on purpose
SIZES = {
    "jacobi7": [8, (5, 6, 9), (33, 47, 70)],
    "wave4": [6, (5, 4, 7), (19, 22, 61)],
    "d3q19": [5, (3, 4, 6), (13, 17, 35)],
    "swim": [12, (9, 14), (131, 257)],
    "clover": [12, (7, 13), (131, 257)],
    "zsolve": [4, (3, 2, 5), (9, 13, 37)],
}


def _torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def to_device(k, name, a, native=True):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if not native:
        return t
    d = backend.empty_native(k, name, tuple(a.shape), t.dtype)   # native strides and start offset
    if d.stride() == t.stride() and d.storage_offset() == 0:
        return t
    backend.copy(d, t)
    return d


def to_host(t):
    torch = _torch()
    if not t.is_contiguous():
        rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
        backend.copy(rm, t)
        t = rm
    torch.cuda.synchronize()
    return t.cpu().numpy()


def run_gpu(kid, ins, scalars, variant, schedule, native=True):
    k = backend.Kernel.lookup(kid)
    dev = {n: to_device(k, n, a, native) for n, a in ins.items()}
    k.launch(dev, scalars, variant, schedule)
    return {n: to_host(t) for n, t in dev.items()}


def bitwise_equal(a, b):
    if a.dtype.kind == "f":
        u = np.uint64 if a.itemsize == 8 else np.uint32
        return np.array_equal(a.view(u), b.astype(a.dtype).view(u))
    return np.array_equal(a, b)


def cases():
    out = []
    for kid, spec in nests.KERNELS.items():
        for size in SIZES[spec.nest]:
            out.append((kid, size))
    return out


def schedules(kid, prec=0):
    """Every registered schedule slot (0 = naive, 1.. = tiled configurations)."""
    k = backend.Kernel.lookup(kid)
    return [i for i, name in enumerate(k.info["schedules"][prec]) if name]


@pytest.mark.parametrize("kid,size", cases(), ids=[f"{k.split(':')[1]}-{s}" for k, s in cases()])
@pytest.mark.parametrize("variant", VARIANTS)
def test_parity_bitexact_vs_oracle(kid, size, variant):
    spec = nests.kernel(kid)
    w = nests.workload(kid, size)
    ins = nests.make_inputs(w)
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(spec, want, w.scalars, variant, fma=variant in SAT)
    for sched in schedules(kid):
        got = run_gpu(kid, ins, w.scalars, variant, sched)
        for n in w.write_arrays:
            assert bitwise_equal(got[n], want[n]), \
                f"{kid} {variant}/{sched} size={size}: '{n}' differs from the oracle " \
                f"(max abs {np.max(np.abs(got[n] - want[n]))})"
        for n in w.read_arrays:
            if n not in w.write_arrays:
                assert bitwise_equal(got[n], ins[n]), f"{kid}: read-only array '{n}' was modified"


@pytest.mark.parametrize("size", [6, (19, 22, 61)])
@pytest.mark.parametrize("variant", VARIANTS)
def test_wave4_fp32_parity(size, variant):
    kid = "wave4.c:wave4:0"
    spec = nests.kernel(kid)
    w = nests.workload(kid, size, dtype="f32")
    ins = nests.make_inputs(w)
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(spec, want, w.scalars, variant, fma=variant in SAT, f32=True)
    for sched in schedules(kid, prec=1):
        got = run_gpu(kid, ins, w.scalars, variant, sched)
        assert bitwise_equal(got["un"], want["un"]), f"wave4 fp32 {variant}/{sched} differs"
    # against the fp64 text: rel 1e-5 with a norm-wise floor
    w64 = nests.workload(kid, size)
    ins64 = {n: a.astype(np.float64) for n, a in ins.items()}
    ref = {n: a.copy() for n, a in ins64.items()}
    oracle_cpu.run(spec, ref, w64.scalars, "original")
    d = np.abs(got["un"].astype(np.float64) - ref["un"])
    floor = 1e-5 * np.max(np.abs(ref["un"]))
    assert np.all((d <= 1e-5 * np.maximum(np.abs(ref["un"]), np.abs(got["un"]))) | (d <= floor))


VEC = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "vectors", "*.npz")))


@pytest.mark.parametrize("path", VEC, ids=[os.path.basename(p)[:-4] for p in VEC])
@pytest.mark.parametrize("variant", VARIANTS)
def test_gpu_vs_reference_interpreter(path, variant):
    """Directly against the reference's own executor (golden vectors)."""
    z = np.load(path)
    fn = os.path.basename(path).split(".")[0]
    spec = nests.kernel(fn)
    scalars = json.loads(bytes(z["scalars"]).decode())
    ins = {k[3:]: (z[k].astype(np.int32) if z[k].dtype.kind == "i" else z[k]) for k in z.files if k.startswith("in_")}
    got = run_gpu(spec.kernel_id, ins, scalars, variant, "default")
    for key in z.files:
        if not key.startswith(f"out_{variant}_"):
            continue
        name = key[len(f"out_{variant}_"):]
        want = z[key]
        if variant in SAT:
            d = np.abs(got[name] - want)
            mag = np.maximum(np.abs(got[name]), np.abs(want))
            assert np.all((d <= 1e-12 * mag) | (d <= 1e-12)), f"{fn}/{variant}/{name}"
        else:
            assert bitwise_equal(got[name], want), f"{fn}/{variant}/{name} differs from the reference interpreter"


def test_rowmajor_and_native_layouts_agree():
    kid = "d3q19.c:stream_collide:0"
    w = nests.workload(kid, (7, 9, 12))
    ins = nests.make_inputs(w)
    a = run_gpu(kid, ins, w.scalars, "accsat", "default", native=True)
    b = run_gpu(kid, ins, w.scalars, "accsat", "default", native=False)
    assert bitwise_equal(a["dst"], b["dst"])


def test_device_fill_matches_host_inputs():
    torch = _torch()
    for kid in ("d3q19.c:stream_collide:0", "clover.c:pdv_predict:1", "wave4.c:wave4:0"):
        for dt in (("f64", "f32") if "wave4" in kid else ("f64",)):
            w = nests.workload(kid, (5, 6, 7) if "clover" not in kid else (9, 11), dtype=dt)
            ins = nests.make_inputs(w)
            k = backend.Kernel.lookup(kid)
            for p in w.spec.arrays:
                fl = w.fills[p.name]
                if fl.kind == "copy":
                    continue
                tdt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32}[ins[p.name].dtype.type]
                t = backend.empty_native(k, p.name, ins[p.name].shape, tdt)
                lo = fl.value if fl.kind == "const" else fl.lo
                backend.fill(t, fl.kind, nests.SEED_BASE + p.position, lo, fl.hi, fl.p)
                assert bitwise_equal(to_host(t), ins[p.name]), f"{kid}:{p.name}"


def test_tune_picks_a_registered_slot_and_keeps_parity():
    kid = "jacobi7.c:jacobi7:0"
    w = nests.workload(kid, (20, 33, 70))
    ins = nests.make_inputs(w)
    k = backend.Kernel.lookup(kid)
    dev = {n: to_device(k, n, a) for n, a in ins.items()}
    best, ms = k.tune(dev, dict(w.scalars), "accsat", reps=2)
    assert best in ms and len(ms) == len(schedules(kid))
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(w.spec, want, w.scalars, "accsat", fma=True)
    got = run_gpu(kid, ins, w.scalars, "accsat", "default")
    assert bitwise_equal(got["Anext"], want["Anext"])


def test_errors_are_loud():
    kid = "jacobi7.c:jacobi7:0"
    w = nests.workload(kid, 6)
    ins = nests.make_inputs(w)
    k = backend.Kernel.lookup(kid)
    dev = {n: to_device(k, n, a) for n, a in ins.items()}
    bad = dict(w.scalars, kend=w.scalars["kend"] + 1)   # would read A0[k+1] past the end
    with pytest.raises(backend.EvalError):
        k.launch(dev, bad, "accsat")
    with pytest.raises(backend.EvalError):
        k.launch({"A0": dev["A0"]}, w.scalars, "accsat")
    with pytest.raises(backend.EvalError):
        backend.Kernel.lookup("nope.c:f:0")


@pytest.mark.parametrize("kid,size,dtype", [("d3q19.c:stream_collide:0", (13, 9, 20), "f64"),
                                            ("jacobi7.c:jacobi7:0", (21, 9, 33), "f64"),
                                            ("swim.c:calc1:0", (37, 65), "f64"),
                                            ("clover.c:advec_cell_x:2", (29, 45), "f64"),
                                            ("wave4.c:wave4:0", (17, 8, 33), "f32")])
@pytest.mark.parametrize("chunks", [1, 3, 5])
def test_host_runner_overlapped_equals_oracle(kid, size, dtype, chunks):
    """The overlapped host-buffer path (chunked H2D | kernel | D2H) gives the
    single-launch result bit for bit."""
    torch = _torch()
    from paper_2306_13002_b200 import pipeline_exec
    spec = nests.kernel(kid)
    w = nests.workload(kid, size, dtype=dtype)
    ins = nests.make_inputs(w)
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(spec, want, w.scalars, "accsat", fma=True, f32=dtype == "f32")
    host = {n: torch.from_numpy(a.copy()).pin_memory() for n, a in ins.items()}
    k = backend.Kernel.lookup(kid)
    r = pipeline_exec.HostRunner(k, host, spec.range_params, chunks=chunks)
    # poison the device staging: elements the shell-only upload skips must be
    # overwritten by the launch, never read
    for n in ins:
        for t in (r.rm[n], r.nat[n]):
            t.fill_(float("nan") if t.dtype.is_floating_point else -12345)
    r.run(dict(w.scalars), "accsat")
    torch.cuda.synchronize()
    for n in ins:
        assert bitwise_equal(host[n].numpy(), want[n]), f"{kid} chunks={chunks}: '{n}'"
    # a second call on fresh inputs reuses the buffers and the shell plan
    ins2 = {n: (a * a.dtype.type(0.75) if a.dtype.kind == "f" else a.copy()) for n, a in ins.items()}
    want2 = {n: a.copy() for n, a in ins2.items()}
    oracle_cpu.run(spec, want2, w.scalars, "accsat", fma=True, f32=dtype == "f32")
    for n in ins2:
        host[n].copy_(torch.from_numpy(ins2[n]))
    r.run(dict(w.scalars), "accsat")
    torch.cuda.synchronize()
    for n in ins2:
        assert bitwise_equal(host[n].numpy(), want2[n]), f"{kid} chunks={chunks} (second call): '{n}'"


@pytest.mark.parametrize("kid,size,dtype", [("d3q19.c:stream_collide:0", (13, 9, 20), "f64"),
                                            ("wave4.c:wave4:0", (17, 8, 33), "f32")])
def test_host_runner_graph_replay_equals_oracle(kid, size, dtype):
    """The host-buffer call captured as a CUDA graph: replaying it on new host
    inputs (same buffers) gives the oracle's result for those inputs."""
    torch = _torch()
    from paper_2306_13002_b200 import pipeline_exec
    spec = nests.kernel(kid)
    w = nests.workload(kid, size, dtype=dtype)
    ins = nests.make_inputs(w)
    host = {n: torch.from_numpy(a.copy()).pin_memory() for n, a in ins.items()}
    k = backend.Kernel.lookup(kid)
    r = pipeline_exec.HostRunner(k, host, spec.range_params, chunks=3)
    g = r.capture(dict(w.scalars), "accsat")
    ins2 = {n: (a * a.dtype.type(0.5) if a.dtype.kind == "f" else a.copy()) for n, a in ins.items()}
    want = {n: a.copy() for n, a in ins2.items()}
    oracle_cpu.run(spec, want, w.scalars, "accsat", fma=True, f32=dtype == "f32")
    for n in ins2:
        host[n].copy_(torch.from_numpy(ins2[n]))
    g.replay()
    torch.cuda.synchronize()
    for n in ins2:
        assert bitwise_equal(host[n].numpy(), want[n]), f"{kid} graph replay: '{n}'"


@pytest.mark.parametrize("kid,size", cases(), ids=[f"{k.split(':')[1]}-{s}" for k, s in cases()])
def test_original_nvcc_default_within_tolerance(kid, size):
    """ACS_ORIGINAL_NVCC (measurement baseline: the original text with nvcc's
    default contraction) agrees with the reference's two-rounding original
    within rel 1e-12 or a norm-wise floor 1e-12 * max|ref|."""
    spec = nests.kernel(kid)
    w = nests.workload(kid, size)
    ins = nests.make_inputs(w)
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(spec, want, w.scalars, "original")
    got = run_gpu(kid, ins, w.scalars, "original-nvcc", 0)
    for n in w.write_arrays:
        a, b = got[n].astype(np.float64), want[n].astype(np.float64)
        if got[n].dtype.kind != "f":
            assert np.array_equal(a, b), f"{kid} original-nvcc: integer array '{n}' differs"
            continue
        d = np.abs(a - b)
        floor = 1e-12 * np.max(np.abs(b)) if b.size else 0.0
        ok = (d <= 1e-12 * np.maximum(np.abs(a), np.abs(b))) | (d <= floor)
        assert np.all(ok), f"{kid} original-nvcc size={size}: '{n}' max abs {np.max(d)}"


def test_cpp_host_api_on_gpu():
    """The C++ host API end to end (tests/cpp/host_api_check.cpp): eval_region
    of jacobi7 original + accsat bit-exact vs a C++ restatement, comparator
    rule, EvalError on a missing array."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "host_api_check")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(root, "tests", "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "host_api_check ok" in r.stdout, r.stdout + r.stderr


# ---- edge cases: empty iteration spaces ---------------------------------------

@pytest.mark.parametrize("kid", sorted(nests.KERNELS))
@pytest.mark.parametrize("which", ["outer", "inner"])
def test_empty_iteration_space_is_a_noop(kid, which):
    """A nest whose loop range is empty (kbeg == kend, or no interior rows)
    runs no point: every array keeps its input bits, in every form and
    schedule slot (the interpreter executes zero iterations)."""
    spec = nests.kernel(kid)
    dtype = "f32" if spec.nest == "wave4" else "f64"
    w = nests.workload(kid, {3: (4, 5, 9), 2: (6, 9)}[len(spec.loop_vars)], dtype=dtype)
    sc = dict(w.scalars)
    beg, end = spec.range_params
    if which == "outer":
        sc[end] = sc[beg]
    else:
        key = "ny" if "ny" in sc and len(spec.loop_vars) == 3 else "nx"
        sc[key] = 1             # every inner loop bound (n - 1, n - 2) is then empty
    ins = nests.make_inputs(w)
    for variant in VARIANTS:
        for sched in schedules(kid, prec=1 if dtype == "f32" else 0):
            got = run_gpu(kid, ins, sc, variant, sched)
            for n in ins:
                assert bitwise_equal(got[n], ins[n]), f"{kid} {variant}/{sched} empty {which}: '{n}' changed"

# Full BASELINE sizes (every form, naive + tuned slots, wave4 1024^3, zsolve 256^3,
# the Jacobi graph step, the slab path, the e2e path) and edge values: tests/test_gpu_fullsize.py


def test_host_runner_byte_mask():
    """D3Q19's 0/1 flags held on the host as bytes (the kernel reads int32):
    the host-buffer call widens them on the device, same result."""
    torch = _torch()
    from paper_2306_13002_b200 import pipeline_exec
    kid = "d3q19.c:stream_collide:0"
    spec = nests.kernel(kid)
    w = nests.workload(kid, (9, 7, 20))
    ins = nests.make_inputs(w)
    want = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(spec, want, w.scalars, "accsat", fma=True)
    host = {n: torch.from_numpy(a.astype(np.uint8) if n == "flags" else a.copy()).pin_memory() for n, a in ins.items()}
    r = pipeline_exec.HostRunner(backend.Kernel.lookup(kid), host, spec.range_params, chunks=3)
    r.run(dict(w.scalars), "accsat")
    torch.cuda.synchronize()
    assert bitwise_equal(host["dst"].numpy(), want["dst"])
    assert r.bytes_per_call()[0] < sum(a.nbytes for a in ins.values())


@pytest.mark.parametrize("size", [(6, 7, 19), (21, 9, 70), (33, 47, 130)])
@pytest.mark.parametrize("nsteps", [1, 2, 5, 8])
@pytest.mark.parametrize("variant", ["original", "accsat"])
def test_temporal_blocking_equals_step_by_step(size, nsteps, variant):
    """acs_launch_steps with temporal blocking (two Jacobi sweeps per launch,
    the step-1 field held in shared memory) gives the newest field of the
    ping-pong time loop bit for bit (odd counts end with one plain step)."""
    torch = _torch()
    kid = "jacobi7.c:jacobi7:0"
    spec = nests.kernel(kid)
    w = nests.workload(kid, size)
    ins = nests.make_inputs(w)
    g = {n: a.copy() for n, a in ins.items()}
    for t in range(nsteps):
        roles = nests.role_buffers(spec.nest, list(g), t)
        oracle_cpu.run(spec, {p: g[b] for p, b in roles.items()}, w.scalars, variant, fma=variant in SAT)
    newest = nests.role_buffers(spec.nest, list(g), nsteps)["A0"]
    k = backend.Kernel.lookup(kid)
    dev = {n: to_device(k, n, a) for n, a in ins.items()}
    latest = k.launch_steps(dev, dict(w.scalars), variant, nsteps, blocked=True)
    got = to_host(dev[latest])
    assert bitwise_equal(got, g[newest]), f"{size} x{nsteps}"


@pytest.mark.parametrize("size", [(6, 7, 13), (21, 9, 70), (33, 47, 130), (70, 40, 37), (230, 12, 37)])
@pytest.mark.parametrize("nsteps", [2, 4, 6])
@pytest.mark.parametrize("variant", ["original", "accsat"])
def test_wave4_leapfrog2_equals_step_by_step(size, nsteps, variant):
    """acs_launch_leapfrog2 (two wave4 fp32 steps per launch, kernels/tbwave.cuh:
    step 1 to un, step 2 to a fourth buffer) rotated like the time loop gives the
    newest u and up of the step-by-step oracle bit for bit.  Precondition of the
    two-step launch (as for Jacobi's): every rotating buffer carries the same
    fixed boundary (the time loop's boundary condition) — set here from u's."""
    torch = _torch()
    kid = "wave4.c:wave4:0"
    spec = nests.kernel(kid)
    w = nests.workload(kid, size, dtype="f32")
    ins = nests.make_inputs(w)
    sc = w.scalars
    inner = np.zeros(ins["u"].shape, dtype=bool)
    inner[int(sc["kbeg"]):int(sc["kend"]), 2:int(sc["ny"]) - 2, 2:int(sc["nx"]) - 2] = True
    for n in ("up", "un"):
        ins[n][~inner] = ins["u"][~inner]
    g = {n: a.copy() for n, a in ins.items()}
    for t in range(nsteps):
        roles = nests.role_buffers(spec.nest, list(g), t)
        oracle_cpu.run(spec, {p: g[b] for p, b in roles.items()}, w.scalars, variant, fma=variant in SAT, f32=True)
    roles = nests.role_buffers(spec.nest, list(g), nsteps)
    k = backend.Kernel.lookup(kid)
    dev = {n: to_device(k, n, a) for n, a in ins.items()}
    x = to_device(k, "un", ins["un"])        # the fourth buffer: any content (un's layout)
    bufs = {"u": dev["u"], "up": dev["up"], "un": dev["un"], "x": x}
    for _ in range(nsteps // 2):
        k.launch_leapfrog2({"u": bufs["u"], "up": bufs["up"], "un": bufs["un"], "vel2": dev["vel2"]}, bufs["x"],
                           dict(w.scalars), variant)
        bufs = {"u": bufs["x"], "up": bufs["un"], "un": bufs["up"], "x": bufs["u"]}
    assert bitwise_equal(to_host(bufs["u"]), g[roles["u"]]), f"{size} x{nsteps}: u"
    assert bitwise_equal(to_host(bufs["up"]), g[roles["up"]]), f"{size} x{nsteps}: up"
    assert bitwise_equal(to_host(dev["vel2"]), ins["vel2"])
