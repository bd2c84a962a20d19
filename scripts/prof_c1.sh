#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
if python scripts/c3_profile.py 1 > gpurun_out/c1_plain.log 2>&1; then
  timeout 900 $NCU -k 'regex:k_kron<' -s 40 -c 1 -o gpurun_out/r02_c1_passA python scripts/c3_profile.py 1 > gpurun_out/ncu_c1a.log 2>&1
  timeout 900 $NCU -k 'regex:k_stream<\(int\)0, \(bool\)0>' -s 40 -c 1 -o gpurun_out/r02_c1_passB python scripts/c3_profile.py 1 > gpurun_out/ncu_c1b.log 2>&1
fi
if python scripts/c3_profile.py 3 > gpurun_out/c3_plain.log 2>&1; then
  timeout 900 $NCU -k 'regex:k_stream<\(int\)0, \(bool\)0>' -s 20 -c 1 -o gpurun_out/r02_c3_passB_v2 python scripts/c3_profile.py 3 > gpurun_out/ncu_c3b2.log 2>&1
fi
echo done
