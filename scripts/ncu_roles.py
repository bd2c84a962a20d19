"""Development aid: stall samples of an ncu report grouped by execution count (= warp role in a warp-specialised
kernel) with the top stall reasons, then the hottest SASS lines with their two main reasons."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
nlines = int(sys.argv[2]) if len(sys.argv) > 2 else 20
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, data = rows[1], rows[2:]
H = {h: i for i, h in enumerate(hdr)}
sc, ex, al = H["Source"], H["Instructions Executed"], H["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(x[al] or 0) for x in data)
grp = defaultdict(lambda: defaultdict(float))
for x in data:
    e = int(x[ex] or 0)
    for h in stalls:
        grp[e][h] += float(x[H[h]] or 0)
    grp[e]["_all"] += float(x[al] or 0)
    grp[e]["_n"] += 1
for e, d in sorted(grp.items(), key=lambda kv: -kv[1]["_all"])[:8]:
    top = sorted(((v, k) for k, v in d.items() if k.startswith("stall_")), reverse=True)[:6]
    print(f"exec={e:>9d} n={int(d['_n']):4d} samples {100 * d['_all'] / tot:5.1f}% :",
          ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for v, k in top))
print()
for x in sorted(data, key=lambda x: -float(x[al] or 0))[:nlines]:
    top = sorted(((float(x[H[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{100 * float(x[al]) / tot:5.1f}% {x[ex]:>9s} {x[sc][:70]:70s} {top[0][1]}:{top[0][0]:.0f} {top[1][1]}:{top[1][0]:.0f}")
