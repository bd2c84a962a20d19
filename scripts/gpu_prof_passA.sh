#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 1500 $NCU -k 'regex:k_kron_mma<\(bool\)0>' -s 60 -c 1 -f -o gpurun_out/r02_c4_passA_v2 $B > gpurun_out/ncu_a.log 2>&1
echo rc=$?
