#!/bin/bash
# round-2 evidence at c4: full GPU test suite, the default bench line, the launch list and ncu captures of the passes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu --timeout 1200 --durations=10 > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
python bench.py > gpurun_out/r02_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02_bench.log
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-witness --no-trace-all"
if $B > gpurun_out/b1.log 2>&1; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
  timeout 1500 $NCU -k 'regex:k_stream<\(int\)0, \(bool\)1>' -s 60 -c 1 -o gpurun_out/r02_c4_passB $B > gpurun_out/ncu_b.log 2>&1
  timeout 1500 $NCU -k 'regex:k_stream<\(int\)1, \(bool\)1>' -s 60 -c 1 -o gpurun_out/r02_c4_passC $B > gpurun_out/ncu_c.log 2>&1
  timeout 1500 $NCU -k 'regex:k_kron_mma<\(bool\)0>' -s 60 -c 1 -o gpurun_out/r02_c4_passA $B > gpurun_out/ncu_a.log 2>&1
fi
echo done
