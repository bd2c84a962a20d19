#!/bin/bash
# GPU test subset (development aid): pytest -m gpu with an optional -k expression
cd "$GRAFT_REPO_ROOT" || exit 1
timeout ${2:-1200} python -m pytest tests -m gpu -q ${3:--x} ${1:+-k "$1"} > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -30 gpurun_out/gpu_tests.log
