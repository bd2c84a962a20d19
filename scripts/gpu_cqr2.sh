#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 --durations=8 > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
tail -25 gpurun_out/t_all.log
