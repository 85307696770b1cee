"""The B200 wrapper hand-off (paper_2306_13002_b200/jit.py) — host side.

satcc's wrapper mode (proj/tools/satcc_main.cpp:285-360) with this backend as
the downstream: stubs replace the nest functions by acs_eval_host calls, the
file's kernels are built into a library exporting the same C ABI, files that
do not parse pass through, the child's exit code comes back."""
import ctypes
import os
import subprocess
import sys

import pytest

from paper_2306_13002_b200 import jit
from paper_2306_13002_b200 import kernel_subset as ks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEAT = os.path.join(ROOT, "tests", "jit", "heat.c")


def test_stub_replaces_the_nest_function():
    src = open(HEAT).read()
    text, ids = jit.stub_source(src, "heat.c", "accsat")
    assert ids == ["heat.c:heat:0"]
    assert '#include "accsat_b200.h"' in text and "acs_eval_host" in text
    assert 'acs_jit_run_("heat.c:heat:0", ACS_ACCSAT, a_, 3, s_, 5);' in text
    assert "for (j = jbeg" not in text          # the loops left for the GPU
    # the stub compiles as C against the ABI header
    p = os.path.join(ROOT, "build", "jit_stub_check.c")
    os.makedirs(os.path.dirname(p), exist_ok=True)
    open(p, "w").write(text)
    r = subprocess.run(["gcc", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), p], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_region_among_other_statements_is_launched_in_place():
    """Statements outside the region stay on the host; the region becomes a launch where it was."""
    src = """void f(double a[8], double b[8]) {
    int i;
    a[0] = 1.0;
    #pragma acc parallel loop gang
    for (i = 0; i < 8; i++) {
        b[i] = a[i] * 2.0;
    }
    a[1] = b[3];
}
"""
    mod = ks.parse(src)
    regs = ks.find_regions(mod)
    assert not jit.offloadable(mod.functions[0], regs)          # not the whole function ...
    assert jit.offload_regions(mod, mod.functions[0], regs) == regs   # ... but the region in place
    text, ids = jit.stub_source(src, "f.c", "accsat")
    assert ids == ["f.c:f:0"] and "a[0] = 1.0;" in text and "a[1] = b[3];" in text
    assert "for (i = 0" not in text and text.index("a[0] = 1.0;") < text.index("acs_jit_run_(\"f.c:f:0\"")


def test_region_with_a_live_out_scalar_stays_on_the_cpu():
    src = """void f(double a[8], double b[8]) {
    int i;
    double s;
    #pragma acc parallel loop gang
    for (i = 0; i < 8; i++) {
        s = a[i] * 2.0;
        b[i] = s;
    }
    a[0] = s;
}
"""
    text, ids = jit.stub_source(src, "f.c", "accsat")
    assert ids == [] and "for (i = 0" in text


def test_time_loop_regions_take_the_loop_index_and_live_ins():
    """An unmarked loop enclosing the regions stays on the host: each region is
    launched per iteration with the loop index (t) and the live-in local (w)
    as scalars (lowering.region_view); the stub compiles against the ABI."""
    from paper_2306_13002_b200 import lowering
    path = os.path.join(ROOT, "tests", "jit", "tloop.c")
    src = open(path).read()
    mod = ks.parse(src)
    r0, r1 = ks.find_regions(mod)
    _, _, imp0 = lowering.region_view(mod, r0.function, r0)
    _, _, imp1 = lowering.region_view(mod, r1.function, r1)
    assert [p.name for p in imp0] == ["t", "w"] and [p.name for p in imp1] == ["t"]
    low = lowering.lower_text(src, "relax", False, region_index=0)
    assert low.loop_vars == ["j", "i"] and "t" in [p.name for p in low.params]
    text, ids = jit.stub_source(src, "tloop.c", "accsat")
    assert ids == ["tloop.c:relax:0", "tloop.c:relax:1"]
    assert "for (t = 0; t < nt; t++)" in text and "for (j = 1" not in text
    assert '{"t", 1, t, 0.0}' in text and '{"w", 0, 0, w}' in text
    p = os.path.join(ROOT, "build", "jit_stub_tloop.c")
    os.makedirs(os.path.dirname(p), exist_ok=True)
    open(p, "w").write(text)
    r = subprocess.run(["gcc", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), p], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_function_bodies_spans():
    src = "/* void g() { */\nvoid f(double a[2]) { int i; { } }\nvoid h(int n) {\n}\n"
    spans = jit._function_bodies(src)
    assert set(spans) == {"f", "h"}
    b, e = spans["f"]
    assert src[b] == "{" and src[e - 1] == "}" and src[b:e] == "{ int i; { } }"


def test_wrap_propagates_exit_code_and_passes_unparseable_files():
    assert jit.wrap([sys.executable, "-c", "import sys; sys.exit(3)"]) == 3
    bad = os.path.join(ROOT, "build", "not_subset.c")
    os.makedirs(os.path.dirname(bad), exist_ok=True)
    open(bad, "w").write("#include <stdio.h>\nint main(void) { return 0; }\n")
    # the unparseable file reaches the child unchanged (its path is not substituted)
    code = "import sys; sys.exit(0 if sys.argv[1] == %r else 9)" % bad
    assert jit.wrap([sys.executable, "-c", code, bad]) == 0


def test_jit_library_builds_and_registers():
    """nvcc builds the file's kernels with the backend's C ABI; the library
    exports every entry point and registers the region under its key."""
    lib, ids = jit.build(HEAT)
    L = ctypes.CDLL(lib)
    assert ids == ["heat.c:heat:0"]
    assert L.acs_kernel_count() == 1
    L.acs_kernel_id.restype = ctypes.c_char_p
    assert L.acs_kernel_id(0) == b"heat.c:heat:0"
    for sym in ("acs_lookup", "acs_launch", "acs_eval_host", "acs_tune", "acs_launch_sharded"):
        assert hasattr(L, sym)
