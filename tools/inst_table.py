#!/usr/bin/env python3
"""Builds the instruction / global-load evidence table (north star: "the
instruction count and global-load count before and after saturation") from
an ncu metrics pass over tools/gpu/inst_evidence.py:

    python tools/inst_table.py gpurun_out/inst_plan.json gpurun_out/inst_metrics.csv > profiles/<round>_instructions.md
"""
import csv
import json
import sys

plan = json.load(open(sys.argv[1]))
rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
iid, mn, mv, kn = (hdr.index(x) for x in ("ID", "Metric Name", "Metric Value", "Kernel Name"))
per = {}
for r in data:
    d = per.setdefault(int(r[iid]), {"kernel": r[kn]})
    d[r[mn]] = float(r[mv].replace(",", ""))
print("# Instruction and global-load evidence, original vs saturated (ncu, B200)\n")
print("Per interior point (thread-level: warp instructions x 32 / points). `static` = the reference's "
      "`count_static_loads` of the form (metrics JSON); `LDG` = global load instructions executed "
      "(nvcc still CSEs identical loads inside a statement); `LDS` = shared-memory loads of the tiled "
      "skeletons, which replace LDGs; `FMA` = extracted single-rounding FMAs; DRAM/alg = measured "
      "dram bytes over algorithmic bytes. Sizes: jacobi 256^3, d3q19 128^3, swim/clover 4096^2, wave4 512^3 f32.\n")
print("| nest | form | skeleton | static loads | FMA | inst/pt | LDG/pt | STG/pt | LDS/pt | DRAM/alg | kernel |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for i, p in enumerate(plan):
    m = per.get(i, {})
    pts = p["points"]
    g = lambda k: m.get(k, float("nan")) * 32 / pts
    dram = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / p["algorithmic_bytes"]
    print(f"| {p['kernel'].split(':')[1]} | {p['variant']} | {p['schedule']} | {p['static_loads']} | {p['fma']} | "
          f"{g('smsp__inst_executed.sum'):.1f} | {g('smsp__inst_executed_op_global_ld.sum'):.2f} | "
          f"{g('smsp__inst_executed_op_global_st.sum'):.2f} | {g('smsp__inst_executed_op_shared_ld.sum'):.2f} | "
          f"{dram:.3f} | `{m.get('kernel', '')[:48]}` |")
