#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cholqr2 or tsqr or solve_parity" > gpurun_out/t_cqr.log 2>&1
echo "cqr tests rc=$?"; tail -3 gpurun_out/t_cqr.log
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k 'regex:k_cqr_pass' -c 3 --log-file gpurun_out/cqr_c4_launches.csv $B > gpurun_out/ncu_cqr_c4.log 2>&1
python - <<'PY'
import csv
f="gpurun_out/cqr_c4_launches.csv"
rows=[r for r in csv.reader(l for l in open(f) if l.startswith('"'))]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value"); mi=hdr.index("Metric Name")
for r in rows[1:]:
    print(r[ki][:40], r[mi][:40], r[vi])
PY
