"""Development aid: warp-stall samples of an ncu report grouped by (execution count, opcode)."""
import csv, subprocess, sys, re
from collections import defaultdict
rep=sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, data = rows[1], rows[2:]
si, sc, ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(float(x[si] or 0) for x in data) or 1.0
agg=defaultdict(float); cnt=defaultdict(int)
for x in data:
    e=int(float(x[ex] or 0)); op=x[sc].split()[0] if x[sc].split() else ''
    if op.startswith('@'): op=x[sc].split()[1]
    key=(e, op.split('.')[0])
    agg[key]+=float(x[si] or 0); cnt[key]+=1
for k,v in sorted(agg.items(), key=lambda kv:-kv[1])[:30]:
    print(f"{100*v/tot:5.1f}%  exec={k[0]:>10d}  {k[1]:12s} n={cnt[k]}")
