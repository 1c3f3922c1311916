#!/bin/bash
# Full round-2 GPU session: pytest -m gpu, smoke, B200 calibration of the
# layout selector, default bench + reference arm, ncu evidence.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash scripts/gpu_r2.sh test
timeout 600 build/tools/calibrate_b200 gpurun_out/b200_calibration.txt > gpurun_out/r02_calibration_log.txt 2>&1
bash scripts/gpu_r2.sh bench
bash scripts/gpu_ncu_r2.sh ${NCU_WHAT:-vgg softmax pl5 transform alexnet}
echo done
