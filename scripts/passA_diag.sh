#!/bin/bash
# Development aid: pass A time with parts of k_kron_mma switched off (diagnostic builds, wrong results):
# $1 = extra nvcc flags, e.g. "-DKM_DIAG_NO_EPI"
cd "$GRAFT_REPO_ROOT" || exit 1
IFS=',' read -ra LIST <<< "${DIAGS:-,-DKM_DIAG_NO_EPI,-DKM_DIAG_NO_MATH,-DKM_DIAG_NO_EL,-DKM_DIAG_NO_EPI -DKM_DIAG_NO_EL}"
for f in "${LIST[@]}"; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr $f -I include -o paper_2510_14471_b200/libglsgpu.so paper_2510_14471_b200/csrc/glsgpu.cu || exit 1
  timeout 600 python bench.py --no-cpu --no-e2e --steps 1 --warmup 2 > gpurun_out/pd.log 2>&1
  tail -1 gpurun_out/pd.log | tee -a gpurun_out/pd_all.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$f]', d.get('iterations'), {k:round(v['avg_ms'],3) for k,v in d['passes'].items()})"
done
