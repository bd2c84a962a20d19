#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -m gpu --timeout 900 -x > gpurun_out/t_quick.log 2>&1
echo "quick rc=$?" >> gpurun_out/t_quick.log
python scripts/config_times.py --only 1,3 --out gpurun_out/r02_config_times_b.jsonl > gpurun_out/config_times_b.log 2>&1
python bench.py --steps 2 --warmup 2 --no-cpu --no-witness > gpurun_out/bench_short2.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_short2.log
