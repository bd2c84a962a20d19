#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -m gpu --timeout 900 > gpurun_out/t_q.log 2>&1; tail -3 gpurun_out/t_q.log
for v in wy lc; do
  GLSGPU_QR_FORMQ=$v python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all > gpurun_out/qrv_$v.log 2>&1
  echo "formq=$v $(grep -o '"setup_qr_ms": [0-9.]*' gpurun_out/qrv_$v.log) $(grep -o '"value": [0-9.]*' gpurun_out/qrv_$v.log | head -1)"
done
B="python bench.py --rows 200000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
if $B > gpurun_out/b200k.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launch_wy.csv -k regex:k_qr $B > gpurun_out/ncu_ql.log 2>&1
fi
