"""The CPU oracle (oracle/, test infrastructure) pinned against the REFERENCE.

Golden vectors in tests/golden/vectors were produced by the reference's own
interpreter (eval_region, proj/src/interp.cpp:266-270) through
tools/gen_vectors.py.  The compiled-C oracle must reproduce them BIT-EXACTLY
for the original text and for every reference-emitted variant (two-rounding
forms), like the reference's own bitwise fidelity tests
(proj/tests/test_codegen.cpp:519-532, proj/tests/test_pipeline.cpp:170-190).
"""
import glob
import json
import os

import numpy as np
import pytest

import cpu as oracle_cpu
from paper_2306_13002_b200 import nests

VEC_DIR = os.path.join(os.path.dirname(__file__), "golden", "vectors")
VECTORS = sorted(glob.glob(os.path.join(VEC_DIR, "*.npz")))
VARIANTS = ["original", "cse", "cse+sat", "cse+bulk", "accsat"]


def load(path):
    z = np.load(path)
    fn = os.path.basename(path).split(".")[0]
    spec = nests.kernel(fn)
    scalars = json.loads(bytes(z["scalars"]).decode())
    ins = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    outs = {k[4:]: z[k] for k in z.files if k.startswith("out_")}
    return spec, scalars, ins, outs


REF_TOOL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "ref_tool")


def _same_extraction(spec, variant):
    """Our stage (a) objective equals the reference optimizer's for this region."""
    from paper_2306_13002_b200 import stage_a
    ours = stage_a.metrics(spec.nest, variant)["regions"][spec.region]["objective_after"]
    ref = json.load(open(os.path.join(nests.GOLDEN_DIR, f"{spec.nest}.{variant}.json")))
    return ours == ref["regions"][spec.region]["objective_after"]


def _ref_eval(spec, variant, scalars, ins):
    """The reference's eval_region over our emitted text (oracle/_ref/ref_tool eval)."""
    import subprocess
    import tempfile
    import envio
    from paper_2306_13002_b200 import stage_a
    with tempfile.TemporaryDirectory() as td:
        ein, eout = os.path.join(td, "in.bin"), os.path.join(td, "out.bin")
        sc = {p.name: (p.ctype, scalars[p.name]) for p in spec.scalars}
        envio.write_env(ein, sc, {k: np.ascontiguousarray(v) for k, v in ins.items()})
        r = subprocess.run([REF_TOOL, "eval", stage_a.emitted_path(spec.nest, variant), spec.function, ein, eout],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        return envio.read_env(eout)[1]


def test_vectors_present():
    assert len(VECTORS) == 2 * len(nests.KERNELS)


@pytest.mark.parametrize("path", VECTORS, ids=[os.path.basename(p)[:-4] for p in VECTORS])
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("text", ["stage_a", "reference"])
def test_oracle_matches_reference_interpreter(path, variant, text):
    """Both emitted texts — host stage (a)'s (what the GPU runs) and the
    reference optimizer's — compiled by gcc give the reference interpreter's
    results bit for bit (two-rounding FMA, as the interpreter evaluates it)."""
    spec, scalars, ins, outs = load(path)
    arrays = {k: np.ascontiguousarray(v.astype(np.int32) if v.dtype.kind == "i" else v.copy())
              for k, v in ins.items()}
    oracle_cpu.run(spec, arrays, scalars, variant, ref=text == "reference")
    if text == "stage_a" and variant in ("cse+sat", "accsat") and not _same_extraction(spec, variant):
        # our exact extraction found a strictly cheaper selection than the reference's
        # (reassociated sums round differently): pin it with the reference interpreter
        # run live on OUR emitted text (oracle/_ref, built from /root/reference)
        if not os.path.exists(REF_TOOL):
            pytest.skip("strictly cheaper extraction: needs oracle/_ref (the reference interpreter)")
        outs = {f"{variant}_{k}": v for k, v in _ref_eval(spec, variant, scalars, ins).items()}
    prefix = f"{variant}_"
    checked = 0
    for key, want in outs.items():
        if not key.startswith(prefix):
            continue
        name = key[len(prefix):]
        got = arrays[name]
        assert got.shape == want.shape
        assert np.array_equal(got.view(np.uint64), want.astype(np.float64).view(np.uint64)), \
            f"{spec.function}/{variant}/{name} differs bitwise from the reference interpreter"
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("path", VECTORS[:4], ids=[os.path.basename(p)[:-4] for p in VECTORS[:4]])
def test_oracle_omp_driver_equals_serial(path):
    spec, scalars, ins, outs = load(path)
    a1 = {k: np.ascontiguousarray(v.astype(np.int32) if v.dtype.kind == "i" else v.copy()) for k, v in ins.items()}
    a2 = {k: v.copy() for k, v in a1.items()}
    oracle_cpu.run(spec, a1, scalars, "accsat")
    oracle_cpu.run(spec, a2, scalars, "accsat", threads=3)
    for k in a1:
        assert np.array_equal(a1[k], a2[k])


@pytest.mark.parametrize("kid,size,dtype", [("jacobi7.c:jacobi7:0", (5, 6, 7), "f64"),
                                            ("d3q19.c:stream_collide:0", (4, 5, 6), "f64"),
                                            ("wave4.c:wave4:0", (6, 5, 9), "f32"),
                                            ("swim.c:calc2:1", (9, 11), "f64"),
                                            ("clover.c:pdv_predict:1", (7, 9), "f64"),
                                            ("zsolve.c:z_solve_lhs:0", (3, 4, 5), "f64")])
def test_host_fill_matches_make_inputs(kid, size, dtype):
    """oracle/fill.c (the reference arm's input generator) is bit-identical to
    nests.make_inputs for every fill kind."""
    w = nests.workload(kid, size, dtype=dtype)
    want = nests.make_inputs(w)
    got = oracle_cpu.host_inputs(w, threads=3)
    assert set(got) == set(want)
    for n in want:
        assert got[n].dtype == want[n].dtype and got[n].shape == want[n].shape, n
        u = {8: np.uint64, 4: np.uint32}[want[n].itemsize]
        assert np.array_equal(got[n].view(u), want[n].view(u)), n


CROSS = [("jacobi7.c:jacobi7:0", (6, 7, 9)), ("d3q19.c:stream_collide:0", (4, 5, 7)), ("swim.c:calc1:0", (9, 11)),
         ("swim.c:calc2:1", (9, 11)), ("swim.c:calc3:2", (9, 11)), ("clover.c:ideal_gas:0", (7, 9)),
         ("clover.c:pdv_predict:1", (7, 9)), ("clover.c:advec_cell_x:2", (7, 9)), ("wave4.c:wave4:0", (6, 5, 9)),
         ("zsolve.c:z_solve_lhs:0", (3, 4, 5))]


@pytest.mark.parametrize("kid,size", CROSS, ids=[c[0].split(":")[1] for c in CROSS])
@pytest.mark.parametrize("variant", ["cse", "cse+bulk", "cse+sat", "accsat"])
@pytest.mark.parametrize("fma", [False, True])
def test_stage_a_forms_compute_what_reference_forms_compute(kid, size, variant, fma):
    """Host stage (a)'s emitted form vs the reference optimizer's emitted form
    of the same VariantConfig, both compiled, on the BASELINE input
    distributions: the CSE-only forms bit for bit (CSE never changes
    arithmetic); the saturated forms within the reference comparator rule
    (rel 1e-12 or abs 1e-12, proj/src/oracle.cpp:12,36) — with real
    single-rounding FMAs (fma=True, what the GPU computes) too."""
    if fma and variant not in ("cse+sat", "accsat"):
        pytest.skip("no FMA in the CSE-only forms")
    spec = nests.kernel(kid)
    w = nests.workload(kid, size)
    ins = nests.make_inputs(w)
    ours = {n: a.copy() for n, a in ins.items()}
    theirs = {n: a.copy() for n, a in ins.items()}
    oracle_cpu.run(spec, ours, w.scalars, variant, fma=fma)
    oracle_cpu.run(spec, theirs, w.scalars, variant, fma=fma, ref=True)
    for n in w.write_arrays:
        a, b = ours[n], theirs[n]
        if variant in ("cse", "cse+bulk"):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), n
        else:
            d = np.abs(a - b)
            assert np.all((d <= 1e-12 * np.maximum(np.abs(a), np.abs(b))) | (d <= 1e-12)), (n, float(d.max()))
