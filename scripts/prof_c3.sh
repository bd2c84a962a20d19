#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
if python scripts/c3_profile.py > gpurun_out/c3_plain.log 2>&1; then
  timeout 1200 $NCU -k 'regex:k_stream<\(int\)0, \(bool\)0>' -s 20 -c 1 -o gpurun_out/r02_c3_passB python scripts/c3_profile.py > gpurun_out/ncu_c3b.log 2>&1
  timeout 1200 $NCU -k 'regex:k_stream<\(int\)1, \(bool\)0>' -s 20 -c 1 -o gpurun_out/r02_c3_passC python scripts/c3_profile.py > gpurun_out/ncu_c3c.log 2>&1
fi
echo done
