"""The benchmark nests: registration keys, parameter lists and seeded workloads.

Each nest is a kernel-subset C file under ``nests/`` (the ORIGINAL form); the
reference optimizer's output for it is frozen under ``tests/golden/emitted/``.
A *kernel id* is ``"<file>:<function>:<region index>"`` — the key
``find_regions`` (proj/src/ast.cpp:390-398) gives each region, in source order
across the module.

Parameters are discovered by parsing the nest text (``kernel_subset``): array
parameters keep the reference layout (row-major, ``ArrayBuf::flat``,
proj/src/interp.cpp:10-22), scalar parameters are ``int``/``double``
(``Scalar``, proj/include/satcc/interp.hpp:13-24).  Loop bounds are scalar
parameters, so one registered kernel serves every grid size.

Synthetic inputs: every array element is drawn from a
counter-based SplitMix64 stream — seed ``20261017 + parameter position``,
counter = flat element index — mapped to ``lo + (hi - lo) * u`` with
``u = (x >> 11) * 2**-53`` (two roundings, no contraction).  The identical
generator runs on the GPU (``acs_fill_uniform``), so full-size workloads are
produced in HBM without a host copy and small ones are bit-identical on both
sides.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import kernel_subset as ks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NEST_DIR = os.path.join(ROOT, "nests")
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden", "emitted")

SEED_BASE = 20261017
VARIANTS = ("original", "cse", "cse+sat", "cse+bulk", "accsat")


@dataclass
class ParamSpec:
    name: str
    ctype: str                 # 'double' | 'int'
    dims: Tuple[int, ...]      # () for scalars; the nest text's declared dims
    position: int


@dataclass
class KernelSpec:
    nest: str                  # file stem, e.g. "swim"
    function: str
    region: int                # find_regions index within the module
    params: List[ParamSpec]
    loop_vars: List[str]       # marked loops, outermost first (GPU iteration space)
    range_params: Tuple[str, str]   # scalar params bounding the outermost loop

    @property
    def kernel_id(self) -> str:
        return f"{self.nest}.c:{self.function}:{self.region}"

    @property
    def arrays(self) -> List[ParamSpec]:
        return [p for p in self.params if p.dims]

    @property
    def scalars(self) -> List[ParamSpec]:
        return [p for p in self.params if not p.dims]


def _load_specs() -> Dict[str, KernelSpec]:
    out = {}
    for nest in ("jacobi7", "swim", "clover", "wave4", "d3q19", "zsolve"):
        with open(os.path.join(NEST_DIR, f"{nest}.c")) as f:
            mod = ks.parse(f.read())
        for reg in ks.find_regions(mod):
            fn = reg.function
            params = [ParamSpec(p.name, p.ty, tuple(p.dims), i) for i, p in enumerate(fn.params)]
            outer = reg.loops[0]
            rng = (outer.init.rhs.op, outer.cond.kids[1].op)
            spec = KernelSpec(nest, fn.name, reg.index, params,
                              [l.loop_var for l in reg.marked_loops], rng)
            out[spec.kernel_id] = spec
    return out


KERNELS: Dict[str, KernelSpec] = _load_specs()


def kernel(kernel_id_or_function: str) -> KernelSpec:
    if kernel_id_or_function in KERNELS:
        return KERNELS[kernel_id_or_function]
    for k in KERNELS.values():
        if k.function == kernel_id_or_function:
            return k
    raise KeyError(kernel_id_or_function)


# ---------------------------------------------------------------------------
# Seeded inputs

_M64 = (1 << 64) - 1


def splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based SplitMix64: the (idx+1)-th output of the stream seeded
    with `seed`.  uint64 arithmetic wraps."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int, lo: float, hi: float, offset: int = 0) -> np.ndarray:
    x = splitmix64(seed, np.arange(offset, offset + n, dtype=np.uint64))
    u = (x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return np.float64(lo) + np.float64(hi - lo) * u


@dataclass
class Fill:
    """How one array is initialised: uniform [lo, hi), a copy of another
    array, a Bernoulli(p) 0/1 mask (int arrays), D3Q19 equilibrium-ish
    weights, or a constant."""
    kind: str = "uniform"
    lo: float = 0.0
    hi: float = 1.0
    src: str = ""
    p: float = 0.0
    value: float = 0.0


D3Q19_W = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)


@dataclass
class Workload:
    """Sizes, scalars and fills of one nest function at one grid size."""
    spec: KernelSpec
    dims: Dict[str, Tuple[int, ...]]
    scalars: Dict[str, float]
    fills: Dict[str, Fill]
    dtype: str = "f64"                      # f64 | f32 (wave4 fp32 config)
    points: int = 0                         # interior points per sweep
    bytes_per_point: int = 0                # algorithmic bytes
    read_arrays: List[str] = field(default_factory=list)
    write_arrays: List[str] = field(default_factory=list)

    @property
    def algorithmic_bytes(self) -> int:
        return self.points * self.bytes_per_point


def _grid3(n):
    return (n, n, n) if isinstance(n, int) else tuple(n)


def workload(kernel_id: str, size=None, dtype: str = "f64") -> Workload:
    """The BASELINE.json / SURVEY.md §8d workload of one nest function.

    `size` is the interior extent (int, or (nz, ny, nx) / (ny, nx) tuple for
    ragged grids); None = the BASELINE config size."""
    s = kernel(kernel_id)
    f = s.function
    esz = 4 if dtype == "f32" else 8
    if s.nest == "jacobi7":
        nz, ny, nx = _grid3(size or 256)
        d = (nz + 2, ny + 2, nx + 2)
        dims = {"A0": d, "Anext": d}
        sc = {"c0": 1.0 / 6.0, "c1": 1.0 / 36.0, "kbeg": 1, "kend": nz + 1, "ny": d[1], "nx": d[2]}
        fills = {"A0": Fill("uniform", 0.0, 1.0), "Anext": Fill("copy", src="A0")}
        return Workload(s, dims, sc, fills, "f64", nz * ny * nx, 16, ["A0"], ["Anext"])
    if s.nest == "wave4":
        nz, ny, nx = _grid3(size or 1024)
        d = (nz + 4, ny + 4, nx + 4)
        dims = {a: d for a in ("u", "up", "un", "vel2")}
        sc = {"c0": -7.5, "c1": 4.0 / 3.0, "c2": -1.0 / 12.0, "kbeg": 2, "kend": nz + 2,
              "ny": d[1], "nx": d[2]}
        fills = {"u": Fill("uniform", -1e-3, 1e-3), "up": Fill("uniform", -1e-3, 1e-3),
                 "un": Fill("const", value=0.0), "vel2": Fill("uniform", 0.05, 0.15)}
        return Workload(s, dims, sc, fills, dtype, nz * ny * nx, 4 * esz,
                        ["u", "up", "vel2"], ["un"])
    if s.nest == "d3q19":
        nz, ny, nx = _grid3(size or 256)
        d = (nz + 2, ny + 2, nx + 2)
        dims = {"src": d + (19,), "dst": d + (19,), "flags": d}
        sc = {"omega": 1.95, "zbeg": 1, "zend": nz + 1, "ny": d[1], "nx": d[2]}
        fills = {"src": Fill("d3q19", -0.01, 0.01), "dst": Fill("d3q19", -0.01, 0.01),
                 "flags": Fill("mask", p=0.1)}
        # 19 reads + 19 writes of 8 B + the 1-byte flag of SURVEY §8d (the device keeps the
        # nest's int32 flags, so 3 B/point moved are not credited — DESIGN Next 2)
        return Workload(s, dims, sc, fills, "f64", nz * ny * nx, 19 * 8 * 2 + 1,
                        ["src", "flags"], ["dst"])
    if s.nest == "swim":
        ny, nx = (size, size) if isinstance(size, int) else (size or (8192, 8192))
        d = (ny + 1, nx + 1)
        names = [a.name for a in s.arrays]
        dims = {a: d for a in names}
        tdt = 90.0 * 2
        allsc = {"fsdx": 4.0 / 1e5, "fsdy": 4.0 / 1e5, "tdts8": tdt / 8.0, "tdtsdx": tdt / 1e5,
                 "tdtsdy": tdt / 1e5, "alpha": 0.001, "jbeg": 0, "jend": ny, "nx": d[1]}
        sc = {p.name: allsc[p.name] for p in s.scalars}
        fills = {}
        for a in names:
            if a.startswith("p"):
                fills[a] = Fill("uniform", 49000.0, 51000.0)
            elif a in ("u", "v", "uold", "vold", "unew", "vnew"):
                fills[a] = Fill("uniform", -20.0, 20.0)
            else:
                fills[a] = Fill("uniform", -1.0, 1.0)
        rw = {"calc1": (["u", "v", "p"], ["cu", "cv", "z", "h"]),
              "calc2": (["uold", "vold", "pold", "cu", "cv", "z", "h"], ["unew", "vnew", "pnew"]),
              "calc3": (["u", "v", "p", "uold", "vold", "pold", "unew", "vnew", "pnew"],
                        ["uold", "vold", "pold", "u", "v", "p"])}[f]
        bpp = {"calc1": 56, "calc2": 80, "calc3": 120}[f]
        return Workload(s, dims, sc, fills, "f64", ny * nx, bpp, rw[0], rw[1])
    if s.nest == "clover":
        ny, nx = (size, size) if isinstance(size, int) else (size or (7680, 7680))
        d = (ny + 4, nx + 4)
        dims = {a.name: (d if len(a.dims) == 2 else (d[1],)) for a in s.arrays}
        allsc = {"dt": 0.04, "one_by_six": 1.0 / 6.0, "kbeg": 2, "kend": ny + 2, "nx": d[1]}
        sc = {p.name: allsc[p.name] for p in s.scalars}
        table = {"density": (0.2, 1.0), "density0": (0.2, 1.0), "density1": (0.2, 1.0),
                 "energy": (1.0, 2.5), "energy0": (1.0, 2.5), "energy1": (1.0, 2.5),
                 "pressure": (0.5, 1.5), "soundspeed": (0.0, 1.0), "viscosity": (0.0, 0.01),
                 "xvel0": (-0.1, 0.1), "yvel0": (-0.1, 0.1), "vol_flux_x": (-0.1, 0.1),
                 "pre_vol": (1.0, 1.1), "volume_change": (0.0, 1.0), "mass_flux_x": (0.0, 1.0),
                 "ener_flux": (0.0, 1.0)}
        fills = {}
        for a in dims:
            if a in ("volume", "xarea", "yarea", "vertexdx"):
                fills[a] = Fill("const", value=1.0)
            else:
                lo, hi = table[a]
                fills[a] = Fill("uniform", lo, hi)
        rw = {"ideal_gas": (["density", "energy"], ["pressure", "soundspeed"]),
              "pdv_predict": (["xarea", "yarea", "volume", "density0", "energy0", "pressure",
                               "viscosity", "xvel0", "yvel0"],
                              ["volume_change", "energy1", "density1"]),
              "advec_cell_x": (["vol_flux_x", "pre_vol", "density1", "energy1"],
                               ["mass_flux_x", "ener_flux"])}[f]
        bpp = 8 * (len(rw[0]) + len(rw[1]))
        return Workload(s, dims, sc, fills, "f64", ny * nx, bpp, rw[0], rw[1])
    if s.nest == "zsolve":
        # NPB-BT z_solve LHS.  Scalars as BT class-style constants (dt = 0.0008,
        # tz1 = 1/dz^2, tz2 = 1/(2 dz) for dz = 1/(n+1); dz1..dz5 the BT
        # dissipation coefficients); jacobians ~ U[-1, 1].
        nz, ny, nx = _grid3(size or 256)
        g = (nz + 2, ny + 2, nx + 2)
        dims = {"fjacZ": (5, 5) + g, "njacZ": (5, 5) + g, "lhsZ": (5, 5, 3) + g}
        h = 1.0 / (nz + 1)
        sc = {"dt": 0.0008, "tz1": 1.0 / (h * h), "tz2": 1.0 / (2.0 * h), "dz1": 1.0, "dz2": 1.0, "dz3": 1.0,
              "dz4": 1.0, "dz5": 1.0, "kbeg": 1, "kend": nz + 1, "ny": g[1], "nx": g[2]}
        fills = {"fjacZ": Fill("uniform", -1.0, 1.0), "njacZ": Fill("uniform", -1.0, 1.0),
                 "lhsZ": Fill("const", value=0.0)}
        # 25 + 25 reads (each element once) + 75 writes of 8 B per point
        return Workload(s, dims, sc, fills, "f64", nz * ny * nx, 8 * 125, ["fjacZ", "njacZ"], ["lhsZ"])
    raise KeyError(kernel_id)


def make_inputs(w: Workload) -> Dict[str, np.ndarray]:
    """Host-side inputs of a workload (reference layout, C types: double or
    float arrays; int arrays as int32 — the compiled nest's `int`)."""
    out: Dict[str, np.ndarray] = {}
    fdt = np.float32 if w.dtype == "f32" else np.float64
    for p in w.spec.arrays:
        shape = w.dims[p.name]
        n = int(np.prod(shape))
        fl = w.fills[p.name]
        seed = SEED_BASE + p.position
        if fl.kind == "uniform":
            a = uniform(seed, n, fl.lo, fl.hi).astype(fdt)
        elif fl.kind == "const":
            a = np.full(n, fl.value, dtype=fdt)
        elif fl.kind == "mask":
            a = (uniform(seed, n, 0.0, 1.0) < fl.p).astype(np.int32)
        elif fl.kind == "d3q19":
            a = (np.tile(D3Q19_W, n // 19) * (1.0 + uniform(seed, n, fl.lo, fl.hi))).astype(fdt)
        elif fl.kind == "copy":
            a = out[fl.src].reshape(-1).copy()
        else:
            raise ValueError(fl.kind)
        if p.ctype == "int" and a.dtype != np.int32:
            a = a.astype(np.int32)
        out[p.name] = a.reshape(shape)
    return out


def scalar_values(w: Workload) -> Dict[str, float]:
    return dict(w.scalars)


def device_inputs(w: Workload, native: bool = True, kernel=None, stream=None):
    """Allocates and fills the workload directly in HBM (acs_fill: the same
    SplitMix64 stream as make_inputs, so values are bit-identical).  Arrays
    use the backend's preferred strides when `native`."""
    import torch
    from . import backend
    k = kernel or backend.Kernel.lookup(w.spec.kernel_id)
    tdt = torch.float32 if w.dtype == "f32" else torch.float64
    out = {}
    for p in w.spec.arrays:
        dt = torch.int32 if p.ctype == "int" else tdt
        dims = w.dims[p.name]
        t = backend.empty_native(k, p.name, dims, dt) if native else torch.empty(dims, dtype=dt, device="cuda")
        fl = w.fills[p.name]
        if fl.kind == "copy":
            backend.copy(t, out[fl.src], stream)
        else:
            lo = fl.value if fl.kind == "const" else fl.lo
            backend.fill(t, fl.kind, SEED_BASE + p.position, lo, fl.hi, fl.p, stream)
        out[p.name] = t
    return out


# ---------------------------------------------------------------------------
# Time stepping: the arrays each nest produces and how buffers rotate between
# steps (Jacobi ping-pong, D3Q19 src <-> dst, wave4 up <- u <- un <- up).

ROTATIONS = {
    "jacobi7": [("A0", "Anext")],
    "d3q19": [("src", "dst")],
    "wave4": [("up", "u", "un")],
}


def role_buffers(nest: str, names, step: int) -> Dict[str, str]:
    """Parameter name -> physical buffer name at `step` (0-based)."""
    out = {n: n for n in names}
    for group in ROTATIONS.get(nest, []):
        L = len(group)
        for i, p in enumerate(group):
            out[p] = group[(i + step) % L]
    return out


def rotation_period(nest: str) -> int:
    """Steps after which every buffer is back in its starting role."""
    p = 1
    for group in ROTATIONS.get(nest, []):
        p = p * len(group) // np.gcd(p, len(group))
    return p


def pipeline_inputs(kernel_ids, size=None, dtype: str = "f64"):
    """Host inputs of a multi-kernel step (shard.PIPELINES): the union of the
    kernels' arrays, each filled by the first kernel that declares it (the
    same rule SlabRank uses on the device).  Returns (arrays, workloads)."""
    ws = [workload(k, size, dtype=dtype) for k in kernel_ids]
    out: Dict[str, np.ndarray] = {}
    for w in ws:
        ins = make_inputs(w)
        for p in w.spec.arrays:
            out.setdefault(p.name, ins[p.name])
    return out, ws

