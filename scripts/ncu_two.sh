#!/bin/bash
# ncu --set full of pass B and pass C of the c4 bench (development aid)
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_stream<\(int\)(0|1), " -s 4 -c 2 -o gpurun_out/${1:-passBC} \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${1:-passBC}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${1:-passBC}.log
