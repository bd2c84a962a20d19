#!/bin/bash
# round-2 evidence on one box: per-config timings, then ncu captures of the c3 wide-block passes and the c4 TSQR leaves
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/config_times.py --out gpurun_out/r02_config_times.jsonl > gpurun_out/config_times.log 2>&1
echo "config_times rc=$?" >> gpurun_out/config_times.log
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
if python scripts/c3_profile.py > gpurun_out/c3_plain.log 2>&1; then
  timeout 1200 $NCU -k 'regex:k_stream<0, 0>' -s 5 -c 1 -o gpurun_out/r02_c3_passB python scripts/c3_profile.py > gpurun_out/ncu_c3b.log 2>&1
  timeout 1200 $NCU -k 'regex:k_stream<1, 0>' -s 5 -c 1 -o gpurun_out/r02_c3_passC python scripts/c3_profile.py > gpurun_out/ncu_c3c.log 2>&1
fi
B="python bench.py --rows 200000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness"
if $B > gpurun_out/b200k.log 2>&1; then
  timeout 1200 $NCU -k 'regex:k_qr_factor_lc' -s 0 -c 1 -o gpurun_out/r02_qr_factor $B > gpurun_out/ncu_qrf.log 2>&1
  timeout 1200 $NCU -k 'regex:k_qr_formq_lc' -s 0 -c 1 -o gpurun_out/r02_qr_formq $B > gpurun_out/ncu_qrq.log 2>&1
fi
echo done
