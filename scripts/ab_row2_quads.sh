#!/bin/bash
# VGG conv1_1 (ROW row pairs): quad-chunk TMA stores (512 B per channel run, LCNN_ROW2_PAIRS=3)
# against paired 128-B-row boxes (=1)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/q4
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_conv_gemm.py -x -q -k "vgg or row" > gpurun_out/q4/test.log 2>&1; echo rc=$? >> gpurun_out/q4/test.log
: > gpurun_out/q4/ab.jsonl
for r in 1 2; do for k in 3 1; do
  echo "{\"row2_pairs\": $k}" >> gpurun_out/q4/ab.jsonl
  LCNN_ROW2_PAIRS=$k timeout 600 python bench.py --workload vgg16 --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/q4/ab.jsonl 2>> gpurun_out/q4/err.log
done; done
echo done
