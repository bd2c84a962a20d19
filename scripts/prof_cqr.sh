#!/bin/bash
# per-kernel durations of the CholeskyQR2 setup at c4 (bench inputs) and c3, plus one full ncu capture of each c4 pass
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k 'regex:k_cqr' --log-file gpurun_out/cqr_c4_launches.csv $B > gpurun_out/ncu_cqr_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k 'regex:k_cqr|k_q_relayout|k_rank' --log-file gpurun_out/cqr_c3_launches.csv python scripts/config_times.py --only 3 --out gpurun_out/ct3.jsonl > gpurun_out/ncu_cqr_c3.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
for m in 0 1 2; do
  timeout 1500 $NCU -k "regex:k_cqr_pass<\(int\)32, \(int\)$m>" -c 1 -o gpurun_out/r02_cqr_c4_pass$m $B > gpurun_out/ncu_cqr_p$m.log 2>&1
done
python - <<'PY'
import csv,sys
for f in ("gpurun_out/cqr_c4_launches.csv","gpurun_out/cqr_c3_launches.csv"):
    rows=[r for r in csv.reader(l for l in open(f) if l.startswith('"'))]
    hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value"); ui=hdr.index("Metric Unit")
    print(f)
    for r in rows[1:]:
        print("  ", r[ki][:60], r[vi], r[ui])
PY
