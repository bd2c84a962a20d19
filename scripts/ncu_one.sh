#!/bin/bash
# one ncu --set full capture of a kernel of the c4 bench (development aid): $1 = kernel regex, $2 = out name
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s ${3:-3} -c 1 -o gpurun_out/$2 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu ${4:-} > gpurun_out/$2.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/$2.log
