#!/bin/bash
# one GPU-box call: the new tests first, then the whole -m gpu suite, then a short bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -m gpu -k "sharded or stage or diagnostics_from_q or trace_buffer or failed_refactor or host_sharded" --timeout 900 > gpurun_out/t_new.log 2>&1
echo "new rc=$?" >> gpurun_out/t_new.log
python -m pytest tests -q -m gpu --timeout 1200 --durations=15 > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
python bench.py --steps 2 --warmup 1 > gpurun_out/bench_short.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_short.log
