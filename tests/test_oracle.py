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


def test_vectors_present():
    assert len(VECTORS) == 2 * len(nests.KERNELS)


@pytest.mark.parametrize("path", VECTORS, ids=[os.path.basename(p)[:-4] for p in VECTORS])
@pytest.mark.parametrize("variant", VARIANTS)
def test_oracle_matches_reference_interpreter(path, variant):
    spec, scalars, ins, outs = load(path)
    arrays = {k: np.ascontiguousarray(v.astype(np.int32) if v.dtype.kind == "i" else v.copy())
              for k, v in ins.items()}
    oracle_cpu.run(spec, arrays, scalars, variant)
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
