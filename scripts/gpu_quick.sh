#!/bin/bash
# quick GPU check: a subset of the GPU tests + a short c4 bench per Kronecker mode (development aid)
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "${1:-c4 or sigma or kron or counters or c0}" > gpurun_out/tq.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tq.log
for k in ${2:-fma exact}; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 --kron $k > gpurun_out/bq_$k.log 2>&1
echo "bench $k rc=$?"
tail -1 gpurun_out/bq_$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'iter_ms', round(d['iter_ms'],3), 'setup', round(d['setup_qr_ms'],1), {k:round(v['avg_ms'],3) for k,v in d['passes'].items()}, d['clocks'])"
done
