#!/bin/bash
# quick GPU check: pass-A/Kronecker parity tests + a short c4 bench (development aid)
timeout 600 python -m pytest tests -m gpu -q -x -k "${1:-c4 or sigma or kron or counters or c0}" > gpurun_out/tq.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tq.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/bq.log 2>&1
echo "bench rc=$?"
tail -1 gpurun_out/bq.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'iter_ms', d['iter_ms'], 'setup', d['setup_qr_ms'], {k:round(v['avg_ms'],3) for k,v in d['passes'].items()}, d['clocks'])"
