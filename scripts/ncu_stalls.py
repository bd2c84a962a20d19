"""Development aid: summarise an ncu report -- key throughputs, warp stall ratios, hottest SASS lines."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr, vals = r[0], r[2] if len(r) > 2 else r[1]
keys = ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for h, v in zip(hdr, vals):
    if h in keys:
        print(f"{h:80s} {v}")
    if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
        try:
            if float(v) > 0.1:
                print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', ''):60s} {v}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, data = rows[1], rows[2:]
si, sc, ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(float(x[si] or 0) for x in data) or 1.0
for x in sorted(data, key=lambda x: -float(x[si] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"{100 * float(x[si]) / tot:5.1f}%  {x[ex]:>10s}  {x[sc][:90]}")
