#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "kron or sw_direct or fused or G256" > gpurun_out/t_passA.log 2>&1
echo "passA tests rc=$?"; tail -3 gpurun_out/t_passA.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-trace-all > gpurun_out/bench_passA.log 2>&1
echo "bench rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/bench_passA.log"):
    if l.startswith("{"):
        d=json.loads(l)
        print(d["value"], d["ms_per_step"], d["setup_qr_ms"], d["iter_ms"], {k:round(v["avg_ms"],3) for k,v in d["passes"].items()}, d.get("parity_witness",{}).get("rel_b"), d.get("parity_witness",{}).get("strict"))
PY
