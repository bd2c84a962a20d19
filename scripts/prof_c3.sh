#!/bin/bash
# ncu summaries of config 3's wide-block passes B / C and the n_b <= 128 CholeskyQR2 passes (reports summarised on
# the box and removed: gpurun merges at most 64 MiB back)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
P="python scripts/c3_profile.py"
if $P > gpurun_out/c3_plain.log 2>&1; then
  cap() {
    timeout 900 $NCU -k "regex:$2" $3 -c 1 -f -o gpurun_out/$1 $P > gpurun_out/ncu_$1.log 2>&1
    python scripts/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1.txt 2>&1
    python scripts/ncu_roles.py gpurun_out/$1.ncu-rep 24 >> gpurun_out/$1.txt 2>&1
    rm -f gpurun_out/$1.ncu-rep
  }
  cap r02b_c3_passB 'k_stream<\(int\)0, \(bool\)0>' "-s 20"
  cap r02b_c3_passC 'k_stream<\(int\)1, \(bool\)0>' "-s 20"
  for m in 0 1 2; do cap r02b_cqr_c3_pass$m "k_cqr_pass<\(int\)128, \(int\)$m>" "-s 3"; done
fi
cat gpurun_out/c3_plain.log
echo done
