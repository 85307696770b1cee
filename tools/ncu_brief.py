"""Brief of one ncu report (first kernel): duration, DRAM bytes, issue / pipe utilisation,
occupancy limits and the top pc-sample stall reasons.  usage: python tools/ncu_brief.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
get = {n: (v[i], units[i]) for i, n in enumerate(h)}
for k in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
          "smsp__inst_executed.sum"]:
    if k in get:
        print(f"{k:60s} {get[k][0]} {get[k][1]}")
st = sorted(((int(float(val[0].replace(',', '') or 0)), n) for n, val in get.items()
             if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")), reverse=True)
print("stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {c}" for c, n in st[:8]))
