#!/bin/bash
# Development aid: bench each prebuilt library under gpurun_variants/ (pass times per variant).
cd "$GRAFT_REPO_ROOT" || exit 1
cp paper_2510_14471_b200/libglsgpu.so /tmp/lib_orig.so
for v in gpurun_variants/*.so; do
  cp "$v" paper_2510_14471_b200/libglsgpu.so
  timeout 600 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/var.log 2>&1
  tail -1 gpurun_out/var.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['value'],3), {k:round(v['avg_ms'],3) for k,v in d['passes'].items()})"
done
cp /tmp/lib_orig.so paper_2510_14471_b200/libglsgpu.so
