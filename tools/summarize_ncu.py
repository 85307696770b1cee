#!/usr/bin/env python3
"""Summarises ncu reports (gpurun_out/*.ncu-rep) into profiles/.

    python tools/summarize_ncu.py <out.md> <report.ncu-rep>[=<algorithmic bytes>] ...

For each report: kernel name, duration, DRAM read/write bytes (the
`traffic` figure bench.py puts beside the roofline), DRAM / L2 / L1
throughput, issue-slot use, occupancy, registers and the top stall reasons.
Also merges {kernel short name: dram bytes per launch} into
profiles/traffic.json.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"

DETAILS = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
           "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Block Size",
           "Grid Size", "Dynamic Shared Memory Per Block", "L2 Hit Rate", "Eligible Warps Per Scheduler"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"]


def rows(rep, page):
    out = subprocess.run([NCU, "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def summarize(rep, alg_bytes=None):
    d = rows(rep, "details")
    kernel = d[1][4] if len(d) > 1 else "?"
    det = {}
    for r in d[1:]:
        if len(r) > 14 and r[12] in DETAILS:
            det[r[12]] = f"{r[14]} {r[13]}".strip()
    raw = rows(rep, "raw")
    h, units, v = raw[0], raw[1], raw[2]
    rw = {}
    for m in RAW:
        if m in h:
            i = h.index(m)
            rw[m] = (v[i], units[i])
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    rd = to_bytes(*rw["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in rw else None
    wr = to_bytes(*rw["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in rw else None
    return {"report": os.path.basename(rep), "kernel": kernel, "details": det,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "traffic_bytes": (rd + wr) if rd is not None and wr is not None else None,
            "algorithmic_bytes": alg_bytes,
            "inst_executed": rw.get("smsp__inst_executed.sum", ("?", ""))[0],
            "top_stalls": [f"{n} {x:.2f}" for x, n in stalls[:5]]}


def main():
    out_md = sys.argv[1]
    items = []
    for a in sys.argv[2:]:
        rep, _, alg = a.partition("=")
        items.append(summarize(rep, float(alg) if alg else None))
    lines = [f"# ncu summaries ({os.path.basename(out_md)})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` under gpurun (one GPU, "
             "cold-cache replays: compare shares and traffic, not absolute times).", ""]
    for it in items:
        lines.append(f"## {it['kernel'][:120]}")
        lines.append(f"report `{it['report']}`")
        lines.append("")
        for k, v in it["details"].items():
            lines.append(f"* {k}: {v}")
        if it["traffic_bytes"] is not None:
            t = it["traffic_bytes"]
            lines.append(f"* DRAM traffic: read {it['dram_read_bytes'] / 1e6:.1f} MB + write {it['dram_write_bytes'] / 1e6:.1f} MB "
                         f"= {t / 1e6:.1f} MB per launch" + (f" (algorithmic {it['algorithmic_bytes'] / 1e6:.1f} MB, "
                                                             f"ratio {t / it['algorithmic_bytes']:.3f})" if it["algorithmic_bytes"] else ""))
        lines.append(f"* warp instructions: {it['inst_executed']}")
        lines.append(f"* top stalls (cycles per issued instruction): {', '.join(it['top_stalls'])}")
        lines.append("")
    os.makedirs(os.path.dirname(os.path.abspath(out_md)), exist_ok=True)
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = {}
    if os.path.exists(tj):
        traffic = json.load(open(tj))
    for it in items:
        short = it["kernel"].split("<")[1].split(",")[0].split("::")[-1] if "<" in it["kernel"] else it["kernel"]
        if it["traffic_bytes"] is not None:
            traffic[short] = it["traffic_bytes"]
    with open(tj, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
