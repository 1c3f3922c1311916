#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/q4
timeout 1200 python -m pytest tests/test_gpu_conv_gemm.py tests/test_gpu_fullsize.py tests/test_gpu_net.py -x -q > gpurun_out/q4/test2.log 2>&1; echo rc=$? >> gpurun_out/q4/test2.log
SAN=1 bash scripts/sanitize_r2.sh > /dev/null 2>&1
echo done
