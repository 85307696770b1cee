"""compute-sanitizer over every skeleton (race detection).

tests/sanitize_workload.py launches every registered schedule slot of every
nest on small ragged grids — the TMA march ring with its mbarriers, the
register-window march, the cp.async stream ring, the sliced register queue,
the naive skeleton — plus a 2-slab sharded time loop on one device (peer
write-through stores ordered by device flags, graph-replayed) and the
host-buffer pipeline, and checks each against the CPU oracle.  Here it runs
under memcheck (out-of-bounds / misaligned global and shared accesses),
racecheck (shared-memory hazards) and synccheck (barrier misuse); every tool
must report zero errors.

Some GPU pools close compute-sanitizer (their wrapper prints "compute-sanitizer
is closed on this pool" instead of running the tool).  The test then skips
with that reason; the last clean logs are kept under profiles/r02_sanitizer/.
"""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    assert os.path.exists(SAN), "compute-sanitizer not found"
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_workload.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000, cwd=ROOT)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log"), "w") as f:
        f.write(out)
    if "is closed on this pool" in out and "sanitize workload ok" not in out:
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert "sanitize workload ok" in out, out[-3000:]
    clean = ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck"
             else "ERROR SUMMARY: 0 errors")
    assert r.returncode == 0 and clean in out, out[-3000:]
