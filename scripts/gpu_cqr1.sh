#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x > gpurun_out/t_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/t_parity.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-trace-all > gpurun_out/bench_cqr.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_cqr.log
tail -5 gpurun_out/t_parity.log
tail -3 gpurun_out/bench_cqr.log | cut -c1-1500
