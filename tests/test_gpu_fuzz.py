"""Seeded fuzz of the device path: random ragged grids (odd extents, extents
below / around the tile sizes and a warp) for every nest, every form and
every registered schedule slot, bit-exact against the compiled reference text
(SURVEY.md §8d parity bar).  Deterministic: the sizes come from a fixed seed."""
import os
import random
import sys
import zlib

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
import cpu as oracle_cpu  # noqa: E402
from paper_2306_13002_b200 import backend, nests  # noqa: E402

pytestmark = pytest.mark.gpu

VARIANTS = ["original", "cse", "cse+bulk", "cse+sat", "accsat"]
SAT = {"cse+sat", "accsat"}


def sizes(nest, n=6, seed=20261017):
    rng = random.Random(zlib.crc32(nest.encode()) ^ seed)   # stable across processes
    out = []
    for _ in range(n):
        if nest in ("swim", "clover"):
            out.append((rng.randint(1, 40), rng.choice([1, 3, 31, 33, 127, 129, 255, 257])))
        else:
            out.append((rng.randint(1, 9), rng.randint(1, 19), rng.choice([1, 2, 7, 31, 33, 63, 65, 129, 130])))
    return out


CASES = [(kid, s) for kid, spec in sorted(nests.KERNELS.items()) for s in sizes(spec.nest)]


def bitwise_equal(a, b):
    if a.dtype.kind == "f":
        u = np.uint64 if a.itemsize == 8 else np.uint32
        return np.array_equal(a.view(u), b.astype(a.dtype).view(u))
    return np.array_equal(a, b)


@pytest.mark.parametrize("kid,size", CASES, ids=[f"{k.split(':')[1]}-{s}" for k, s in CASES])
def test_fuzz_every_form_and_slot(kid, size):
    import torch
    assert torch.cuda.is_available()
    spec = nests.kernel(kid)
    dtype = "f32" if spec.nest == "wave4" else "f64"
    prec = 1 if dtype == "f32" else 0
    w = nests.workload(kid, size, dtype=dtype)
    ins = nests.make_inputs(w)
    k = backend.Kernel.lookup(kid)
    slots = [i for i, n in enumerate(k.info["schedules"][prec]) if n]
    for variant in VARIANTS:
        want = {n: a.copy() for n, a in ins.items()}
        oracle_cpu.run(spec, want, w.scalars, variant, fma=variant in SAT, f32=dtype == "f32")
        for slot in slots:
            dev = {}
            for n, a in ins.items():
                t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
                d = backend.empty_native(k, n, tuple(a.shape), t.dtype)
                backend.copy(d, t)
                dev[n] = d
            k.launch(dev, dict(w.scalars), variant, slot)
            for n in w.write_arrays:
                t = dev[n]
                rm = torch.empty(t.shape, dtype=t.dtype, device="cuda")
                backend.copy(rm, t)
                torch.cuda.synchronize()
                got = rm.cpu().numpy()
                assert bitwise_equal(got, want[n]), f"{kid} size={size} {variant} slot {slot}: '{n}' differs"
