#!/bin/bash
# the round's last default bench line and ncu launch list (final commit)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python bench.py > gpurun_out/r02b_bench_final.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02b_bench_final.log
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo done
