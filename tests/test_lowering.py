"""The lowering's exact body transformations, checked on CPU (no GPU needed):
if-conversion of store-symmetric branches, unconditional store targets,
component slicing and the register-window row tables — on the real nests
and on small synthetic texts that must be refused.  The generated headers
under csrc/gen/ must be what the lowering produces now (the .so is built
from them)."""
import os
import re

import pytest

from paper_2306_13002_b200 import lowering

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def emitted(nest, variant):
    return open(os.path.join(ROOT, "tests", "golden", "emitted", f"{nest}.{variant}.c")).read()


def original(nest):
    return open(os.path.join(ROOT, "nests", f"{nest}.c")).read()


def lower(text, fn, fma=True, **kw):
    return lowering.lower_text(text, fn, fma, **kw)


# ---- if-conversion -----------------------------------------------------------

def test_d3q19_bulk_forms_if_converted_original_not():
    for variant in ("accsat", "cse+bulk"):
        low = lower(emitted("d3q19", variant), "stream_collide")
        assert low.body.count("if-converted: both arms store the same 19 elements") == 1
        # one store per pushed element, each a select of the two arms
        assert len(re.findall(r"m\.template st<ARR_dst", low.body)) == 19
        assert len(re.findall(r"\(_ifc \? ", low.body)) == 19
    low = lower(original("d3q19"), "stream_collide", fma=False)
    assert "if-converted" not in low.body          # loads inside the arms: left as is
    assert len(re.findall(r"m\.template st<ARR_dst", low.body)) == 38


def test_if_conversion_off_switch_keeps_branch():
    low = lower(emitted("d3q19", "accsat"), "stream_collide", ifconv=False)
    assert "if-converted" not in low.body
    assert len(re.findall(r"m\.template st<ARR_dst", low.body)) == 38


ASYM = """void f(double a[8][8], double b[8][8], int n) {
    int i, j;
    double t;
    #pragma acc parallel loop gang
    for (i = 1; i < n; i++) {
        #pragma acc loop vector
        for (j = 1; j < n; j++) {
            t = a[i][j];
            if (t > 0.0) {
                b[i][j] = t;
            } else {
                b[i][j - 1] = t;
            }
        }
    }
}
"""

LOADS_IN_ARM = ASYM.replace("b[i][j - 1] = t;", "b[i][j] = a[i][j + 1];")

LIVE_AFTER = """void f(double a[8][8], double b[8][8], int n) {
    int i, j;
    double t, u;
    #pragma acc parallel loop gang
    for (i = 1; i < n; i++) {
        #pragma acc loop vector
        for (j = 1; j < n; j++) {
            t = a[i][j];
            if (t > 0.0) {
                u = t;
                b[i][j] = t;
            } else {
                u = 2.0;
                b[i][j] = 1.0;
            }
            a[i][j] = u;
        }
    }
}
"""


@pytest.mark.parametrize("text", [ASYM, LOADS_IN_ARM, LIVE_AFTER], ids=["different-targets", "load-in-arm",
                                                                       "scalar-live-after"])
def test_if_conversion_refused(text):
    low = lower(text, "f", fma=False)
    assert "if-converted" not in low.body


def test_if_conversion_symmetric_synthetic():
    text = ASYM.replace("b[i][j - 1] = t;", "b[i][j] = 2.0 * t;")
    low = lower(text, "f", fma=False)
    assert "if-converted: both arms store the same 1 elements" in low.body


# ---- unconditional store targets ----------------------------------------------

def test_must_write_d3q19_every_push_both_arms():
    low = lower(emitted("d3q19", "accsat"), "stream_collide")
    targets = sorted(t for t in low.must_write if t[0] == "dst")
    assert len(targets) == 19
    assert {t[1][3] for t in targets} == set(range(19))      # one per component q
    low0 = lower(original("d3q19"), "stream_collide", fma=False)
    assert sorted(low0.must_write) == sorted(low.must_write)


def test_must_write_excludes_one_armed_store():
    low = lower(ASYM, "f", fma=False)
    assert low.must_write == set()                           # each arm writes a different element


# ---- component slicing --------------------------------------------------------

@pytest.mark.parametrize("variant", ["original", "accsat", "cse"])
def test_zsolve_slices_by_block_entry(variant):
    text = original("zsolve") if variant == "original" else emitted("zsolve", variant)
    low = lower(text, "z_solve_lhs", fma=variant == "accsat")
    assert len(low.slices) == 25
    for sl, refs in zip(low.slices, low.slice_refs):
        assert len(re.findall(r"m\.template st<ARR_lhsZ", sl)) == 3
        # one (m, n) field of each jacobian: fjacZ at k-1, k+1; njacZ at k-1, k, k+1
        comps = {(a, o[0], o[1]) for a, o in refs}
        assert len({(m, n) for _, m, n in comps}) == 1
        assert sorted(a for a, _ in refs) == ["fjacZ", "fjacZ", "njacZ", "njacZ", "njacZ"]


@pytest.mark.parametrize("nest,fn", [("d3q19", "stream_collide"), ("jacobi7", "jacobi7"), ("swim", "calc1"),
                                     ("clover", "pdv_predict")])
def test_coupled_bodies_not_sliced(nest, fn):
    low = lower(emitted(nest, "accsat"), fn)
    assert low.slices == []


# ---- register-window rows -----------------------------------------------------

def test_wave4_row_table():
    """13-point star of u + up + vel2: 11 rows, the x-offset range only on
    the centre row of u (-2..2)."""
    hdr = open(os.path.join(ROOT, "paper_2306_13002_b200", "csrc", "gen", "wave4.cuh")).read()
    m = re.search(r"static constexpr int NROW = (\d+);", hdr)
    assert m and int(m.group(1)) == 11
    xlo = re.search(r"row_xlo\(int r\) \{ constexpr int t\[11\] = \{([^}]*)\}", hdr).group(1)
    assert sorted(int(v) for v in xlo.split(",")) == [-2] + [0] * 10


def test_generated_headers_are_current(tmp_path):
    """csrc/gen/*.cuh (what the library is compiled from) == the lowering now."""
    lowering.generate_all(str(tmp_path))
    for f in sorted(os.listdir(tmp_path)):
        want = open(os.path.join(tmp_path, f)).read()
        have = open(os.path.join(ROOT, "paper_2306_13002_b200", "csrc", "gen", f)).read()
        assert have == want, f"{f} is stale: re-run python -m paper_2306_13002_b200.lowering"


def test_value_set_proven_dynamic_loads():
    """advec: donor / downwind take only affine candidates (j-1 or j); the
    upwind clamp `if (upwind > nx - 1) upwind = nx - 1` after `upwind = j + 1`
    can never fire inside `for (j = 2; j < nx - 2; j++)`, so upwind's
    candidates are {j-2, j+1} too -> every dynamic load is ldx_in."""
    low = lower(emitted("clover", "accsat"), "advec_cell_x")
    assert re.search(r"ldx_in<ARR_density1>\(k, donor\)", low.body)
    assert re.search(r"ldx_in<ARR_pre_vol>\(k, donor\)", low.body)
    assert re.search(r"ldx_in<ARR_density1>\(k, upwind\)", low.body)
    assert not re.search(r"ldx<", low.body)


CLAMP = """void f(double a[64], double b[64], int n) {
    int i, u;
    #pragma acc parallel loop gang
    for (i = 1; i < n - LIMIT; i++) {
        u = i + 1;
        if (u > n - 1) {
            u = n - 1;
        }
        b[i] = a[u];
    }
}
"""


def test_dead_guard_needs_the_loop_bound():
    """The clamp is dead only if i + 1 <= n - 1 for every i of the loop."""
    dead = lower(CLAMP.replace("LIMIT", "2"), "f", fma=False)       # i <= n - 3: dead
    assert "ldx_in<ARR_a>(u)" in dead.body
    live = lower(CLAMP.replace("LIMIT", "0"), "f", fma=False)       # i = n - 1 reaches it
    assert "ldx<ARR_a>(u)" in live.body and "ldx_in" not in live.body
