#!/bin/bash
# TAPS row pairs (C_o <= 64): parity, full-size routes, VGG-16 A/B.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/taps2
timeout 900 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "conv" > gpurun_out/taps2/test.log 2>&1; echo "rc=$?" >> gpurun_out/taps2/test.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "conv_routes or vgg16" > gpurun_out/taps2/test_full.log 2>&1; echo "rc=$?" >> gpurun_out/taps2/test_full.log
: > gpurun_out/taps2/ab.jsonl
for r in 1 2; do for k in 1 0; do
  echo "{\"taps2\": $k}" >> gpurun_out/taps2/ab.jsonl
  LCNN_CONV_TAPS2=$k timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/taps2/ab.jsonl 2>> gpurun_out/taps2/err.log
done; done
echo done
