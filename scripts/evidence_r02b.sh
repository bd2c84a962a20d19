#!/bin/bash
# round-2 (second half) evidence at c4: full GPU test suite, the default bench line, per-config times, the launch
# list and ncu captures of pass A (k_kron_mma2), passes B / C and the CholeskyQR2 setup passes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 --durations=10 > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
tail -4 gpurun_out/t_all.log
timeout 1800 python bench.py > gpurun_out/r02b_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02b_bench.log
timeout 900 python scripts/config_times.py --out gpurun_out/r02b_config_times.jsonl > gpurun_out/config_times.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
if timeout 600 $B > gpurun_out/b1.log 2>&1; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
  timeout 900 $NCU -k 'regex:k_stream<\(int\)0, \(bool\)1>' -s 60 -c 1 -f -o gpurun_out/r02b_c4_passB $B > gpurun_out/ncu_b.log 2>&1
  timeout 900 $NCU -k 'regex:k_stream<\(int\)1, \(bool\)1>' -s 60 -c 1 -f -o gpurun_out/r02b_c4_passC $B > gpurun_out/ncu_c.log 2>&1
  timeout 900 $NCU -k 'regex:k_kron_mma2<\(bool\)0' -s 60 -c 1 -f -o gpurun_out/r02b_c4_passA $B > gpurun_out/ncu_a.log 2>&1
  for m in 0 1 2; do
    timeout 900 $NCU -k "regex:k_cqr_pass<\(int\)32, \(int\)$m>" -c 1 -f -o gpurun_out/r02b_cqr_c4_pass$m $B > gpurun_out/ncu_cqr_p$m.log 2>&1
  done
fi
echo done
