#!/bin/bash
# round-2 (second half) evidence at c4: [the full GPU test suite with `tests`,] the default bench line, per-config
# times, the launch list and ncu summaries of pass A (k_kron_mma2), passes B / C and the CholeskyQR2 setup passes.
# The .ncu-rep files are summarised on the box and removed (gpurun merges at most 64 MiB back).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ "$1" = "tests" ]; then
  timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 --durations=10 > gpurun_out/t_all.log 2>&1
  echo "all rc=$?" >> gpurun_out/t_all.log
  tail -4 gpurun_out/t_all.log
fi
timeout 1800 python bench.py > gpurun_out/r02b_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02b_bench.log
timeout 900 python scripts/config_times.py --out gpurun_out/r02b_config_times.jsonl > gpurun_out/config_times.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
if timeout 600 $B > gpurun_out/b1.log 2>&1; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
  cap() {  # name, kernel regex, extra ncu args
    timeout 900 $NCU -k "regex:$2" $3 -c 1 -f -o gpurun_out/$1 $B > gpurun_out/ncu_$1.log 2>&1
    python scripts/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1.txt 2>&1
    python scripts/ncu_roles.py gpurun_out/$1.ncu-rep 16 >> gpurun_out/$1.txt 2>&1
    rm -f gpurun_out/$1.ncu-rep
  }
  cap r02b_c4_passB 'k_stream<\(int\)0, \(bool\)1>' "-s 60"
  cap r02b_c4_passC 'k_stream<\(int\)1, \(bool\)1>' "-s 60"
  cap r02b_c4_passA 'k_kron_mma2<\(bool\)0' "-s 60"
  for m in 0 1 2; do cap r02b_cqr_c4_pass$m "k_cqr_pass<\(int\)32, \(int\)$m>" ""; done
fi
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
echo done
