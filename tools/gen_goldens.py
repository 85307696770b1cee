#!/usr/bin/env python3
"""Freezes the reference optimizer's output for every benchmark nest.

For each nests/<nest>.c and each VariantConfig name (cse, cse+sat, cse+bulk,
accsat — proj/src/pipeline.cpp:97-110) this runs the UNMODIFIED reference
library through oracle/_ref/ref_tool (optimize_source with the CLI defaults,
proj/tools/satcc_main.cpp:37-53: 10000 nodes / 10 s / 10 iters / ilp / 30 s)
and writes

    tests/golden/emitted/<nest>.<variant>.c      emitted module text
    tests/golden/emitted/<nest>.<variant>.json   satcc-metrics-v1 per region

Needs /root/reference (builds oracle/_ref first).  The outputs are committed:
nothing at test or bench time re-runs the reference optimizer.
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NESTS = ["jacobi7", "swim", "clover", "wave4", "d3q19", "zsolve"]
VARIANTS = ["cse", "cse+sat", "cse+bulk", "accsat"]


def run(nest, variant):
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    src = os.path.join(ROOT, "nests", f"{nest}.c")
    out = os.path.join(ROOT, "tests", "golden", "emitted", f"{nest}.{variant}.c")
    met = os.path.join(ROOT, "tests", "golden", "emitted", f"{nest}.{variant}.json")
    r = subprocess.run([tool, "opt", variant, src, out, met], capture_output=True, text=True)
    return nest, variant, r.returncode, r.stderr


def main():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    os.makedirs(os.path.join(ROOT, "tests", "golden", "emitted"), exist_ok=True)
    jobs = [(n, v) for n in NESTS for v in VARIANTS]
    if len(sys.argv) > 1:
        jobs = [(n, v) for (n, v) in jobs if n in sys.argv[1:]]
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        for nest, variant, rc, err in ex.map(lambda a: run(*a), jobs):
            print(f"{nest:8s} {variant:9s} rc={rc} {err.strip()}")


if __name__ == "__main__":
    main()
