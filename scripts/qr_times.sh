#!/bin/bash
# launch list of the setup kernels of one c4 step (development aid)
ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_qr|k_rank" --csv --log-file gpurun_out/qr_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_qr.log 2>&1
echo rc=$?
