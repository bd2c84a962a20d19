#!/bin/bash
# development aid: the pass A / setup parity tests and a short bench line (per-pass times)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "kron or sw_direct or fused or G256 or cholqr2" > gpurun_out/t_quick.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/t_quick.log
timeout 400 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-trace-all > gpurun_out/bench_quick.log 2>&1
echo "bench rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/bench_quick.log"):
    if l.startswith("{"):
        d=json.loads(l)
        print(d["value"], d["ms_per_step"], d["setup_qr_ms"], d["iter_ms"], {k:round(v["avg_ms"],3) for k,v in d["passes"].items()}, d.get("parity_witness",{}).get("rel_b"), d.get("parity_witness",{}).get("strict"))
PY
