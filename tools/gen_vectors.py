#!/usr/bin/env python3
"""Golden input/output vectors from the REFERENCE INTERPRETER.

For every registered nest function, at small (toy and ragged) grid sizes, this
seeds the workload inputs (paper_2306_13002_b200/nests.py), runs the
reference's own executor ``eval_region`` (proj/src/interp.cpp:266-270) over the
whole function body through oracle/_ref/ref_tool, for the original nest text
and for each of the four reference-emitted variants, and commits

    tests/golden/vectors/<function>.<tag>.npz
        in_<array>            inputs (reference layout)
        out_<variant>_<array> post-state of every array the nest writes
        scalars               JSON of the scalar parameters

These pin the CPU oracle (oracle/gen, compiled C) and through it the sm_100a
kernels.  Needs /root/reference (oracle/_ref); the .npz files are what travels.
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2306_13002_b200 import nests  # noqa: E402
import envio  # noqa: E402

TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
OUT_DIR = os.path.join(ROOT, "tests", "golden", "vectors")

SIZES = {
    "jacobi7": {"toy": 8, "ragged": (5, 6, 9)},
    "wave4": {"toy": 6, "ragged": (5, 4, 7)},
    "d3q19": {"toy": 5, "ragged": (3, 4, 6)},
    "swim": {"toy": 12, "ragged": (9, 14)},
    "clover": {"toy": 12, "ragged": (7, 13)},
    "zsolve": {"toy": 4, "ragged": (3, 2, 5)},
}


def eval_ref(text_path, function, scalars, arrays):
    with tempfile.TemporaryDirectory() as td:
        ein, eout = os.path.join(td, "in.bin"), os.path.join(td, "out.bin")
        envio.write_env(ein, scalars, arrays)
        r = subprocess.run([TOOL, "eval", text_path, function, ein, eout], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"{function}: {r.stderr}")
        return envio.read_env(eout)[1]


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    os.makedirs(OUT_DIR, exist_ok=True)
    summary = {}
    for kid, spec in nests.KERNELS.items():
        for tag, size in SIZES[spec.nest].items():
            w = nests.workload(kid, size)
            ins = nests.make_inputs(w)
            sc = {p.name: (p.ctype, w.scalars[p.name]) for p in spec.scalars}
            blob = {f"in_{k}": v for k, v in ins.items()}
            texts = {"original": os.path.join(ROOT, "nests", f"{spec.nest}.c")}
            for v in ("cse", "cse+sat", "cse+bulk", "accsat"):
                texts[v] = os.path.join(nests.GOLDEN_DIR, f"{spec.nest}.{v}.c")
            outs = {}
            for v, path in texts.items():
                res = eval_ref(path, spec.function, sc, ins)
                outs[v] = res
                for a in w.write_arrays:
                    blob[f"out_{v}_{a}"] = res[a].astype(ins[a].dtype)
            same = {v: all(np.array_equal(outs[v][a], outs["original"][a]) for a in w.write_arrays)
                    for v in texts}
            blob["scalars"] = np.frombuffer(json.dumps(w.scalars).encode(), dtype=np.uint8)
            path = os.path.join(OUT_DIR, f"{spec.function}.{tag}.npz")
            np.savez_compressed(path, **blob)
            summary[f"{spec.function}.{tag}"] = {"size": size, "variant_bitwise_equal_original": same}
            print(f"{spec.function:15s} {tag:7s} {str(size):12s} bitwise-equal-to-original: {same}")
    with open(os.path.join(OUT_DIR, "SUMMARY.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
