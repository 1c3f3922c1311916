#!/bin/bash
# TAPS ring shape A/B on VGG-16 (conv1_2, conv2_1, conv2_2): input-box slots 2/3/4.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ni
: > gpurun_out/ni/ab.jsonl
for r in 1 2; do for k in 3 4 2; do
  echo "{\"ni\": $k}" >> gpurun_out/ni/ab.jsonl
  LCNN_TAPS_NI=$k timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/ni/ab.jsonl 2>> gpurun_out/ni/err.log
done; done
LCNN_TAPS_NI=4 timeout 600 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "conv_chwn" > gpurun_out/ni/test.log 2>&1; echo rc=$? >> gpurun_out/ni/test.log
echo done
