#!/usr/bin/env python3
"""Generates oracle/gen/*.c — the CPU oracle.  TEST INFRASTRUCTURE ONLY.

What the oracle is: the reference's own way of running a nest at scale, i.e.
wrapper mode ``satcc -- cc -O3 kernel.c`` (proj/tools/satcc_main.cpp:285-360):
the nest text (original form) or an optimizer's emitted text is handed to a C
compiler.  Two emitted sets are compiled:

  * ``<form>``      the text host stage (a) emitted — this repo's optimizer
                    (paper_2306_13002_b200/emitted/, stage_a.py): the SAME
                    program the sm_100a kernels are lowered from, so GPU and
                    checker run one text;
  * ``ref_<form>``  the text the UNMODIFIED reference optimizer emitted
                    (tests/golden/emitted/<nest>.<variant>.c, frozen by
                    tools/gen_goldens.py): the cross-check that our forms
                    compute what the reference's forms compute.

This script makes only MECHANICAL edits to those texts:

  1. each function is renamed ``<fn>__<form>`` and its fixed-dim array
     parameters become C99 VLA parameters ``double A[][d1][d2]`` so a single
     build serves every size (the body is untouched; loop bounds are already
     scalar parameters in the nest text);
  2. the ``*_fma`` forms rewrite every emitted FMA temp ``_vN = a + b * c;``
     (an extracted Fma node, printed by proj/src/printer.cpp:114-125) into
     ``_vN = fma(b, c, a);`` — one rounding, as the sm_100a kernels compute it;
     the plain forms keep the reference interpreter's two roundings
     (apply_fma, proj/src/interp.cpp:68-70);
  3. fp32 forms (wave4) are the textual ``double -> float``, ``fma -> fmaf``
     copy, compiled with -fsingle-precision-constant (SURVEY.md §7 hard part 3).

plus an ABI shim per function so ctypes can call it, and an OpenMP driver that
splits the outermost (gang) loop range across host threads.

Compiled by ``make -C oracle cpu`` with gcc -O3 -ffp-contract=off (never
-ffast-math) into oracle/_ref/libacs_cpu.so.
"""
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2306_13002_b200 import kernel_subset as ks  # noqa: E402
from paper_2306_13002_b200 import stage_a  # noqa: E402

NESTS = ["jacobi7", "swim", "clover", "wave4", "d3q19", "zsolve"]
F32_NESTS = {"wave4"}
# (form name, source variant or None for the original text, fma rewrite)
FORMS = [("original", None, False), ("cse", "cse", False), ("cse_bulk", "cse+bulk", False),
         ("cse_sat", "cse+sat", False), ("cse_sat_fma", "cse+sat", True),
         ("accsat", "accsat", False), ("accsat_fma", "accsat", True)]
FORMS = FORMS + [("ref_" + f, v, fma) for f, v, fma in FORMS if v is not None]

FMA_RE = re.compile(r"^(\s*)(_v\d+) = ([A-Za-z_]\w*|-?[0-9.][0-9.eE+-]*) \+ "
                    r"([A-Za-z_]\w*|-?[0-9.][0-9.eE+-]*) \* ([A-Za-z_]\w*|-?[0-9.][0-9.eE+-]*);$")
SIG_RE = re.compile(r"^void (\w+)\((.*)\) \{$")


def int_temps(text):
    out = set()
    for m in re.finditer(r"^\s*int (_v[^;]*);", text, re.M):
        out.update(x.strip() for x in m.group(1).split(","))
    return out


def rewrite_fma(text, fname="fma"):
    ints = int_temps(text)
    n = 0
    lines = []
    for line in text.split("\n"):
        m = FMA_RE.match(line)
        if m and m.group(2) not in ints:
            ind, t, a, b, c = m.groups()
            line = f"{ind}{t} = {fname}({b}, {c}, {a});"
            n += 1
        lines.append(line)
    return "\n".join(lines), n


def split_functions(text):
    """Yields (name, signature params text, full function text) per function."""
    lines = text.split("\n")
    i = 0
    while i < len(lines):
        m = SIG_RE.match(lines[i])
        if not m:
            i += 1
            continue
        j = i + 1
        while lines[j] != "}":
            j += 1
        yield m.group(1), m.group(2), "\n".join(lines[i + 1:j])
        i = j + 1


def vla_params(params):
    """'double A[258][258][258], int n' -> (dim params, VLA params, param list)."""
    plist = []
    for p in (x.strip() for x in params.split(",")):
        ty, rest = p.split(" ", 1)
        name = rest.split("[")[0]
        dims = [int(d) for d in re.findall(r"\[(\d+)\]", rest)]
        plist.append((ty, name, dims))
    dim_decls, vla = [], []
    for ai, (ty, name, dims) in enumerate(plist):
        if dims:
            ds = []
            for k in range(1, len(dims)):
                dim_decls.append(f"long _d_{name}_{k}")
                ds.append(f"[_d_{name}_{k}]")
            vla.append(f"{ty} {name}[]" + "".join(ds))
        else:
            vla.append(f"{ty} {name}")
    return dim_decls, vla, plist


def outer_range_params(fname, params, body):
    """Names of the scalar params bounding the outermost (gang) loop."""
    mod = ks.parse(f"void {fname}({params}) {{\n{body}\n}}\n")
    fn = mod.functions[0]
    reg = ks.find_regions(mod)[0]
    outer = reg.loops[0]
    beg = outer.init.rhs
    end = outer.cond.kids[1]
    assert beg.kind == "var" and end.kind == "var", "outer loop bounds must be scalar params"
    return beg.op, end.op


def emit_function(fname, form, params, body, rng):
    dim_decls, vla, plist = vla_params(params)
    sym = f"{fname}__{form}"
    beg, end = rng
    out = []
    out.append(f"static void {sym}__impl({', '.join(dim_decls + vla)}) {{")
    out.append(body)
    out.append("}")
    # ABI shim: a[] array base pointers, d[] dims (8 per array slot),
    # iv[]/dv[] scalar values by parameter position.
    args, dargs = [], []
    for pi, (ty, name, dims) in enumerate(plist):
        if dims:
            for k in range(1, len(dims)):
                dargs.append(f"d[{pi}*8+{k}]")
            args.append(f"a[{pi}]")
        elif ty == "int":
            args.append(f"(int)iv[{pi}]")
        else:
            args.append(f"({ty})dv[{pi}]")
    pos = {name: pi for pi, (_, name, _) in enumerate(plist)}
    call_args = ", ".join(dargs + args)
    out.append(f"void {sym}(void* const* a, const long* d, const long long* iv, const double* dv) {{")
    out.append(f"    {sym}__impl({call_args});")
    out.append("}")
    # OpenMP driver: static split of [beg, end) over nthreads.
    args_omp = [f"(int)b_" if pi == pos[beg] else (f"(int)e_" if pi == pos[end] else a)
                for pi, a in enumerate(args)]
    out.append(f"void {sym}_omp(void* const* a, const long* d, const long long* iv, const double* dv, int nthreads) {{")
    out.append(f"    long long lo = iv[{pos[beg]}], hi = iv[{pos[end]}];")
    out.append("    #pragma omp parallel for num_threads(nthreads) schedule(static)")
    out.append("    for (int t = 0; t < nthreads; ++t) {")
    out.append("        long long b_ = lo + (hi - lo) * t / nthreads, e_ = lo + (hi - lo) * (t + 1) / nthreads;")
    out.append(f"        if (b_ < e_) {sym}__impl({', '.join(dargs + args_omp)});")
    out.append("    }")
    out.append("}")
    return "\n".join(out) + "\n"


def to_f32(text):
    text = re.sub(r"\bdouble\b", "float", text)
    text = re.sub(r"\bfma\(", "fmaf(", text)
    return text


def generate(nest):
    files = {}
    parts = [f"/* GENERATED by oracle/gen_oracle_c.py from nests/{nest}.c, the stage (a) texts\n"
             f" * paper_2306_13002_b200/emitted/{nest}.<variant>.c and the reference-emitted\n"
             f" * tests/golden/emitted/{nest}.<variant>.c (ref_ forms) — TEST INFRASTRUCTURE ONLY.\n"
             " * Bodies are the reference text verbatim; see the generator for the only edits. */\n",
             '#include "acs_cpu.h"\n']
    f32 = [p for p in parts]
    fma_counts = {}
    for form, variant, fma in FORMS:
        if variant is None:
            path = os.path.join(ROOT, "nests", f"{nest}.c")
        elif form.startswith("ref_"):
            path = os.path.join(ROOT, "tests", "golden", "emitted", f"{nest}.{variant}.c")
        else:
            path = stage_a.ensure(nest, variant)
        text = open(path).read()
        text = re.sub(r"/\*.*?\*/\n?", "", text, flags=re.S)
        for fname, params, body in split_functions(text):
            if fma:
                body, n = rewrite_fma(body)
                fma_counts[(fname, form)] = n
            rng = outer_range_params(fname, params, body)
            parts.append(emit_function(fname, form, params, body, rng))
            if nest in F32_NESTS:
                f32.append(emit_function(fname, form + "_f32", to_f32(params), to_f32(body), rng))
    files[f"{nest}.c"] = "\n".join(parts)
    if nest in F32_NESTS:
        files[f"{nest}_f32.c"] = "\n".join(f32)
    return files, fma_counts


HEADER = """/* GENERATED by oracle/gen_oracle_c.py — TEST INFRASTRUCTURE ONLY. */
#pragma once
#include <math.h>
"""


def main():
    gen = os.path.join(HERE, "gen")
    os.makedirs(gen, exist_ok=True)
    with open(os.path.join(gen, "acs_cpu.h"), "w") as f:
        f.write(HEADER)
    for nest in NESTS:
        files, fc = generate(nest)
        for name, text in files.items():
            with open(os.path.join(gen, name), "w") as f:
                f.write(text)
        for (fn, form), n in sorted(fc.items()):
            print(f"{nest:8s} {fn:15s} {form:12s} fma rewrites = {n}")


if __name__ == "__main__":
    main()
