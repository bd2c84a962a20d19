#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu --timeout 1200 --durations=10 > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
python bench.py --steps 2 --warmup 2 > gpurun_out/bench_short.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_short.log
bash scripts/prof_r02.sh
