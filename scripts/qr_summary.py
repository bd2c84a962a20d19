"""Print the setup-kernel launch list written by scripts/qr_times.sh."""
import csv
from collections import OrderedDict
rows = [r for r in csv.reader(open("gpurun_out/qr_launches.csv")) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d = OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = r[vi]
for (i, k), m in d.items():
    print(i, k[:32], {kk.split("__")[1][:24]: v for kk, v in m.items()})
