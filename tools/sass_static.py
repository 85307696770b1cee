#!/usr/bin/env python3
"""Static SASS opcode histogram of every kernel in the backend library
(cuobjdump -sass), for the evidence tables under profiles/:

    python tools/sass_static.py [lib.so] > profiles/r02_sass_static.md

Per kernel (accsat = form 4 and original = form 0 instantiations, plus the
step-ordering kernels): total SASS instructions, global loads / stores,
shared loads (LDS), TMA bulk-tensor loads (UTMALDG), mbarrier ops (SYNCS),
FP64 / FP32 FMA-add-mul, and whether any tensor-core instruction appears
(none should: no nest is a contraction)."""
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2306_13002_b200", "libaccsat_b200.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = {}
cur = None
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and cur:
        funcs[cur][m.group(2)] += 1
names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
rows = []
for (mangled, c), dem in zip(funcs.items(), names):
    short = dem.replace("acs::", "").replace("gen::", "")
    m = re.match(r"void (\w+)<(\w+), (double|float), (\d+)", short)
    if m:
        form = int(m.group(4))
        if form not in (0, 4):
            continue
    elif "ctr_kernel" not in short:
        continue
    tc = sum(v for k, v in c.items() if k.startswith(("HMMA", "UTCMMA", "UTCHMMA", "UTCQMMA", "DMMA", "IMMA")))
    rows.append((short.split("(")[0], sum(c.values()), c["LDG"], c["STG"], c["LDS"], c["UTMALDG"], c["SYNCS"],
                 c["DFMA"] + c["DADD"] + c["DMUL"], c["FFMA"] + c["FADD"] + c["FMUL"], tc))
print("# Static SASS histograms (cuobjdump -sass of libaccsat_b200.so, sm_100a)\n")
print("Form 4 = accsat (reference's default VariantConfig), form 0 = original. Static counts (instructions in the "
      "binary), not executed counts — see the per-nest ncu summaries for those.\n")
print("| kernel | SASS | LDG | STG | LDS | UTMALDG | SYNCS | DFMA/DADD/DMUL | FFMA/FADD/FMUL | tensor-core |")
print("|---|---|---|---|---|---|---|---|---|---|")
for r in sorted(rows):
    print("| `" + r[0] + "` | " + " | ".join(str(x) for x in r[1:]) + " |")
