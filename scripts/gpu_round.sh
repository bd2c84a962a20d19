#!/bin/bash
# one GPU-box call: the targeted tests first, then the whole -m gpu suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py tests/test_gpu_ne.py tests/test_gpu_reduce.py -q -m gpu --timeout 900 > gpurun_out/t_new.log 2>&1
echo "new rc=$?" >> gpurun_out/t_new.log
python -m pytest tests -q -m gpu --timeout 1200 --durations=15 > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
