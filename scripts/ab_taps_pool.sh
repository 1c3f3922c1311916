#!/bin/bash
# VGG conv1_2 -> pool1 as one kernel (TAPS row pairs with the 2x2 max in the epilogue)
# against the two launches (LCNN_TAPS_POOL=0): parity, then alternating VGG-16 forwards.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/tp
timeout 900 python -m pytest tests/test_gpu_conv_pool.py -x -q > gpurun_out/tp/test.log 2>&1; echo rc=$? >> gpurun_out/tp/test.log
: > gpurun_out/tp/ab.jsonl
for r in 1 2; do for k in 1 0; do
  echo "{\"taps_pool\": $k}" >> gpurun_out/tp/ab.jsonl
  LCNN_TAPS_POOL=$k timeout 600 python bench.py --workload vgg16 --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/tp/ab.jsonl 2>> gpurun_out/tp/err.log
done; done
echo done
