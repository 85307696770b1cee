"""The B200 wrapper hand-off end to end: user programs (tests/jit/main*.c)
calling nest files (tests/jit/heat.c: parameter arrays; matmul_g.c: file-scope
arrays, a sequential inner reduction loop, a branch) compiled through
`acs-satcc --backend b200 -- gcc ...` runs the nest on the GPU and prints
the same bits as the program compiled for the CPU (original and CSE forms:
bit-exact; the saturated form within the reference comparator rule)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
J = os.path.join(ROOT, "tests", "jit")
SATCC = os.path.join(ROOT, "paper_2306_13002_b200", "acs-satcc")


def run(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    h, v = r.stdout.split()
    return h, float(v)


PROGRAMS = {"heat": ("main.c", "heat.c"),               # parameters, 2-D stencil, 4 calls
            "matmul": ("main_matmul.c", "matmul_g.c"),    # file-scope arrays, inner reduction loop, branch
            "tloop": ("main_tloop.c", "tloop.c")}         # host time loop enclosing two regions, live-in local


@pytest.mark.parametrize("prog", sorted(PROGRAMS))
@pytest.mark.parametrize("variant", ["original", "cse", "accsat"])
def test_wrapped_program_runs_on_the_b200(prog, variant):
    main, nest = (os.path.join(J, f) for f in PROGRAMS[prog])
    out = os.path.join(ROOT, "build", f"{prog}_{variant.replace('+', '_')}")
    cpu = os.path.join(ROOT, "build", f"{prog}_cpu")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", main, nest, "-o", cpu], check=True)
    r = subprocess.run([SATCC, "--backend", "b200", "--variant", variant, "--", "gcc", "-O2", "-ffp-contract=off",
                        main, nest, "-o", out], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    nm = subprocess.run(["nm", "-D", out], capture_output=True, text=True).stdout
    assert "acs_eval_host" in nm                # the nest runs through the backend, not on the CPU
    want, got = run(cpu), run(out)
    if variant in ("original", "cse"):
        assert got == want
    else:
        assert abs(got[1] - want[1]) <= 1e-12 * abs(want[1])


def test_report_gpu_fields():
    """acs-satcc report --gpu: satcc-metrics-v1 plus each region's B200 run."""
    import json
    r = subprocess.run([SATCC, "report", "--gpu", "--size", "64", os.path.join(ROOT, "nests", "wave4.c"),
                        os.path.join(ROOT, "nests", "swim.c")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    reps = json.loads(r.stdout)
    regions = [g for rep in reps for g in rep["regions"]]
    assert len(regions) == 4 and all(rep["schema"] == "satcc-metrics-v1" for rep in reps)
    for g in regions:
        gpu = g["gpu"]
        assert "error" not in gpu, gpu
        assert gpu["gbs"] > 0 and 0 < gpu["roofline_frac"] < 2 and gpu["schedule"]
        assert gpu["static_loads"] == g["static_loads_after"] and gpu["fma_count"] == g["fma_count"]
        # the saturated form's single-rounding FMAs vs the original's two roundings
        assert gpu["vs_original"]["max_abs"] <= (1e-7 if gpu["dtype"] == "f32" else 1e-8), gpu
