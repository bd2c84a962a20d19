#!/bin/bash
# run the short c4 bench N times (development aid: run-to-run spread of the per-pass times)
for i in $(seq 1 ${1:-2}); do
timeout 600 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/bq$i.log 2>&1
tail -1 gpurun_out/bq$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'iter_ms', round(d['iter_ms'],2), 'setup', round(d['setup_qr_ms'],1), {k:round(v['avg_ms'],3) for k,v in d['passes'].items()}, d['clocks']['sm_mhz'])"
done
