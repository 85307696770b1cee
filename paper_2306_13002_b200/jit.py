"""The B200 as satcc's downstream: wrapper-mode hand-off for any nest file.

satcc's wrapper mode (``satcc -- cc -O3 kernel.c``, proj/tools/satcc_main.cpp:
285-360) writes the optimized text of every ``*.c`` argument to a temporary
directory and runs the wrapped compiler on it.  ``python -m
paper_2306_13002_b200.jit wrap [--variant V] -- cc ... kernel.c ...`` does the
same with this backend as the target, for any file in the kernel subset:

1. **build** — host stage (a) (``satopt``, our C++ optimizer) emits the four
   VariantConfig forms of the file; ``lowering.gen_function`` turns the
   original and emitted forms of every region function into device bodies;
   a generated registration unit gives each region the default skeletons
   (naive, plus the TMA march skeleton when its loads are stageable); nvcc
   links it with the backend's C ABI into ``libaccsat_jit.so`` (cached by
   content hash under ``build/jit/``);
2. **stub** — every function whose body is declarations plus the region
   loops is re-emitted as calls of ``acs_eval_host`` (eval_region for host
   arrays: upload, launch, download) on the function's own parameters;
   functions with other statements stay on the CPU unchanged (satcc's
   fail-open, satcc_main.cpp:329-332), as do files that do not parse;
3. **exec** — the wrapped command runs on the stub files with the include /
   link flags appended; its exit code is returned (128 + signal, 127 if exec
   fails).

The program then runs its nests on the B200.  The benchmark nests use the
prebuilt, tuned ``libaccsat_b200.so``; this path is for everything else."""
from __future__ import annotations

import hashlib
import os
import re
import shutil
import subprocess
import sys
import tempfile
from typing import Dict, List, Optional, Tuple

from . import kernel_subset as ks

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
CACHE = os.path.join(ROOT, "build", "jit")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
VARIANTS = ["cse", "cse+sat", "cse+bulk", "accsat"]
VARIANT_ENUM = {"original": "ACS_ORIGINAL", "cse": "ACS_CSE", "cse+bulk": "ACS_CSE_BULK", "cse+sat": "ACS_CSE_SAT",
                "accsat": "ACS_ACCSAT"}


class JitError(RuntimeError):
    pass


def offload_regions(mod: ks.Module, fn: ks.Function, regions: List[ks.Region]) -> List[ks.Region]:
    """The regions of `fn` the hand-off can run on the B200.  A function that is
    only its nest goes whole (its body becomes one launch); otherwise each
    region is replaced IN PLACE by a launch and the rest of the function —
    enclosing time loops included — stays on the host, passing the enclosing
    loop indices and the live-in locals as scalars (lowering.region_view).  A
    region whose scalar assignments are read elsewhere in the function (a
    live-out) stays on the CPU (fail-open)."""
    from . import lowering
    if len(regions) == 1 and offloadable(fn, regions):
        return regions
    out = []
    for r in regions:
        try:
            lowering.region_view(mod, fn, r)
        except lowering.LowerError:
            continue
        top = r.marked_loops[0]
        _, writes = lowering._stmt_reads_writes(top)
        writes -= {l.loop_var for l in r.marked_loops}
        inside = {id(t) for t in lowering._walk_stmts(top)}
        outside_reads = set()
        for t in lowering._walk_stmts(fn.body):
            if id(t) in inside or t.kind == "block":
                continue
            rd, _ = lowering._stmt_reads_writes(ks.Stmt(t.kind, lhs=t.lhs, rhs=t.rhs, cond=t.cond, call=t.call,
                                                         names=t.names))
            outside_reads |= rd
        if writes & outside_reads:
            continue
        out.append(r)
    return out


def ns_name(fn: ks.Function, r: ks.Region, whole: bool) -> str:
    return fn.name if whole else f"{fn.name}_r{r.index}"


def offloadable(fn: ks.Function, regions: List[ks.Region]) -> bool:
    """The function body is declarations plus the outermost loops of its
    regions (so replacing it by the region launches keeps its semantics)."""
    tops = {id(r.loops[0]) for r in regions}

    def ok(stmts):
        for s in stmts:
            if s.kind == "decl" and all(not d[2] for d in s.names):
                continue
            if s.kind == "for" and id(s) in tops:
                continue
            if s.kind == "empty":
                continue
            if s.kind == "block" and ok(s.stmts):      # `#pragma acc parallel { ... }`
                continue
            return False
        return True
    return ok(fn.body.stmts if fn.body.kind == "block" else [fn.body])


def _digest(src: str) -> str:
    h = hashlib.sha256(src.encode())
    for rel in ("lowering.py", "kernel_subset.py", "csrc/abi.cu", "csrc/registry.hpp", "csrc/acs_device.cuh",
                "csrc/kernels/march.cuh", "csrc/tma.cuh", "host/acs_opt.cpp"):
        with open(os.path.join(HERE, rel), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def build(c_path: str, cache_dir: Optional[str] = None) -> Tuple[str, List[str]]:
    """Compiles the B200 library for one nest file; returns (library path,
    kernel ids of the offloaded regions)."""
    from . import lowering, satopt
    src = open(c_path).read()
    name = os.path.basename(c_path)
    stem = os.path.splitext(name)[0]
    mod = ks.parse(src)
    regions = ks.find_regions(mod)
    by_fn: Dict[str, List[ks.Region]] = {}
    for r in regions:
        by_fn.setdefault(r.function.name, []).append(r)
    plan = []          # (function, region, struct name)
    for f in mod.functions:
        if f.name not in by_fn:
            continue
        regs = offload_regions(mod, f, by_fn[f.name])
        whole = len(by_fn[f.name]) == 1 and offloadable(f, by_fn[f.name])
        plan += [(f, r, ns_name(f, r, whole)) for r in regs]
    if not plan:
        raise JitError(f"{name}: no region function to offload")
    out = os.path.join(cache_dir or CACHE, f"{stem}_{_digest(src)}")
    lib = os.path.join(out, "libaccsat_jit.so")
    ids = [f"{name}:{f.name}:{r.index}" for f, r, _ in plan]
    if os.path.exists(lib):
        return lib, ids
    os.makedirs(out, exist_ok=True)
    sources: Dict[Optional[str], str] = {None: src}
    for v in VARIANTS:
        text, meta = satopt.optimize_source(src, name, v, exact_time_s=satopt.EXACT_TIME_S)
        sources[v] = text
    parts = [f"// GENERATED by paper_2306_13002_b200/jit.py from {name}", "#pragma once",
             "namespace acs { namespace gen {"]
    for f, r, nsn in plan:
        txt, _ = lowering.gen_function(stem, f.name, sources=sources, region_index=r.index, ns_name=nsn)
        parts.append(txt)
    parts.append("}}  // namespace acs::gen")
    with open(os.path.join(out, "gen_jit.cuh"), "w") as fh:
        fh.write("\n".join(parts) + "\n")
    reg = ["// GENERATED by paper_2306_13002_b200/jit.py", '#include "registry.hpp"', '#include "kernels/march.cuh"',
           '#include "gen_jit.cuh"', "namespace acs {", "void register_jit() {"]
    for f, r, nsn in plan:
        reg += ["    {", "        static Entry e;", f'        e.kernel_id = "{name}:{f.name}:{r.index}";',
                f'        e.function = "{f.name}";', f'        describe<gen::{nsn}>(e, "{name}", {r.index});',
                f"        fill_default<gen::{nsn}, double>(e);", "        register_entry(&e);", "    }"]
    reg += ["}", "}  // namespace acs"]
    with open(os.path.join(out, "jit_reg.cu"), "w") as fh:
        fh.write("\n".join(reg) + "\n")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
           "-fPIC", "--expt-relaxed-constexpr", "-diag-suppress", "177,550", "-I", CSRC, "-I", INCLUDE, "-I", out,
           "-DACS_JIT_REGISTRY", "-shared", os.path.join(CSRC, "abi.cu"), os.path.join(out, "jit_reg.cu"),
           "-o", lib + ".tmp", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise JitError(f"nvcc failed for {name}:\n{r.stderr[-4000:]}")
    os.replace(lib + ".tmp", lib)
    return lib, ids


# ---------------------------------------------------------------------------
# host stubs

def _function_bodies(src: str) -> Dict[str, Tuple[int, int]]:
    """name -> (index of the body's '{', index after its '}') of every function
    definition (comments skipped; the kernel subset has no string literals)."""
    code = re.sub(r"/\*.*?\*/", lambda m: " " * len(m.group(0)), src, flags=re.S)
    code = re.sub(r"//[^\n]*", lambda m: " " * len(m.group(0)), code)
    code = re.sub(r"^\s*#[^\n]*", lambda m: " " * len(m.group(0)), code, flags=re.M)
    out = {}
    for m in re.finditer(r"\bvoid\s+(\w+)\s*\(", code):
        depth, i = 1, m.end()
        while depth and i < len(code):
            depth += {"(": 1, ")": -1}.get(code[i], 0)
            i += 1
        j = i
        while j < len(code) and code[j].isspace():
            j += 1
        if j >= len(code) or code[j] != "{":
            continue
        depth, k = 1, j + 1
        while depth and k < len(code):
            depth += {"{": 1, "}": -1}.get(code[k], 0)
            k += 1
        out[m.group(1)] = (j, k)
    return out


def stub_source(src: str, name: str, variant: str) -> Tuple[str, List[str]]:
    """The file with every offloadable region function's body replaced by
    acs_eval_host calls; returns (text, offloaded kernel ids)."""
    from . import lowering
    mod = ks.parse(src)
    regions = ks.find_regions(mod)
    by_fn: Dict[str, List[ks.Region]] = {}
    for r in regions:
        by_fn.setdefault(r.function.name, []).append(r)
    spans = _function_bodies(src)
    dt = {"double": "ACS_F64", "int": "ACS_I32"}
    edits, ids = [], []

    def launch(f, r, ind):
        kid = f"{name}:{f.name}:{r.index}"
        # the function's own parameters, the file's globals, then (in-place regions) the
        # enclosing loop indices and live-in locals
        params = lowering.region_params(mod, f, r)
        arrs = [p for p in params if p.dims]
        scs = [p for p in params if not p.dims]
        a_init = ", ".join("{" + f'"{p.name}", {dt[p.ty]}, {len(p.dims)}, {{{", ".join(str(d) for d in p.dims)}}}, '
                           f"{{0}}, (void*){p.name}" + "}" for p in arrs)
        s_init = ", ".join("{" + f'"{p.name}", {1 if p.ty == "int" else 0}, '
                           f'{p.name if p.ty == "int" else 0}, {p.name if p.ty != "int" else 0.0}' + "}" for p in scs)
        body = ["{", f"{ind}/* {kid}: offloaded to the B200 by paper_2306_13002_b200/jit.py ({variant}) */"]
        body.append(f"{ind}acs_array a_[{max(1, len(arrs))}] = {{{a_init}}};")
        body.append(f"{ind}acs_scalar s_[{max(1, len(scs))}] = {{{s_init}}};")
        body.append(f'{ind}acs_jit_run_("{kid}", {VARIANT_ENUM[variant]}, a_, {len(arrs)}, s_, {len(scs)});')
        ids.append(kid)
        return body

    for f in mod.functions:
        if f.name not in by_fn:
            continue
        if len(by_fn[f.name]) == 1 and offloadable(f, by_fn[f.name]):
            edits.append((spans[f.name], "\n".join(launch(f, by_fn[f.name][0], "    ") + ["}"])))
            continue
        for r in offload_regions(mod, f, by_fn[f.name]):
            top = r.marked_loops[0]
            ls = src.rfind("\n", 0, top.beg) + 1
            ind = src[ls:top.beg] if src[ls:top.beg].strip() == "" else ""
            edits.append(((top.beg, top.end), ("\n" + ind).join(launch(f, r, "    ") + ["}"])))
    out = src
    for (b, e), text in sorted(edits, key=lambda x: -x[0][0]):
        out = out[:b] + text + out[e:]
    head = ("/* GENERATED by paper_2306_13002_b200/jit.py (B200 hand-off) */\n"
            "#include <stdio.h>\n#include <stdlib.h>\n#include <math.h>\n#include \"accsat_b200.h\"\n"
            "static void acs_jit_run_(const char* id, acs_variant v, acs_array* a, int na, acs_scalar* s, int ns) {\n"
            "    const acs_kernel* k;\n"
            "    if (acs_lookup(id, &k) != ACS_OK || acs_eval_host(k, v, a, na, s, ns) != ACS_OK) {\n"
            "        fprintf(stderr, \"accsat-b200: %s: %s\\n\", id, acs_last_error());\n"
            "        exit(70);\n    }\n}\n")
    return head + out, ids


def wrap(argv: List[str], variant: str = "accsat", keep: bool = False) -> int:
    """Runs `argv` with every offloadable *.c argument replaced by its B200 stub
    and the backend's include / link flags appended; returns the exit code."""
    tmp = tempfile.mkdtemp(prefix="accsat-b200-")
    cmd, libdirs = list(argv), []
    try:
        for i, a in enumerate(argv):
            if not a.endswith(".c") or not os.path.isfile(a):
                continue
            src = open(a).read()
            try:
                text, ids = stub_source(src, os.path.basename(a), variant)
                if not ids:
                    continue
                lib, _ = build(a)
            except Exception as e:       # unparseable / unsupported: the file passes through (fail-open)
                print(f"accsat-b200: {a}: left unchanged ({str(e).splitlines()[0][:200]})", file=sys.stderr)
                continue
            d = os.path.join(tmp, str(i))
            os.makedirs(d, exist_ok=True)
            p = os.path.join(d, os.path.basename(a))
            with open(p, "w") as fh:
                fh.write(text)
            cmd[i] = p
            libdirs.append(os.path.dirname(lib))
        if libdirs:
            cmd += ["-I" + INCLUDE]
            for d in dict.fromkeys(libdirs):
                cmd += [os.path.join(d, "libaccsat_jit.so"), "-Wl,-rpath," + d]
            cmd += ["-L/usr/local/cuda/lib64", "-lcudart", "-lm"]
        try:
            r = subprocess.run(cmd)
        except OSError:
            return 127
        return 128 - r.returncode if r.returncode < 0 else r.returncode
    finally:
        if keep:
            print(f"accsat-b200: kept {tmp}", file=sys.stderr)
        else:
            shutil.rmtree(tmp, ignore_errors=True)


def main(argv: List[str]) -> int:
    variant, keep = "accsat", False
    args = list(argv)
    if args and args[0] == "build":
        for a in args[1:]:
            lib, ids = build(a)
            print(lib, " ".join(ids))
        return 0
    if args and args[0] == "wrap":
        args = args[1:]
    while args and args[0] != "--":
        a = args.pop(0)
        if a == "--variant":
            variant = args.pop(0)
        elif a == "--keep":
            keep = True
        else:
            print(f"usage: python -m paper_2306_13002_b200.jit [build file.c | wrap [--variant V] [--keep] -- cmd]",
                  file=sys.stderr)
            return 2
    if not args:
        print("jit wrap: missing '-- cmd'", file=sys.stderr)
        return 2
    return wrap(args[1:], variant, keep)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
