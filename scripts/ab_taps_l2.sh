#!/bin/bash
# TAPS L2 policies on VGG-16: LCNN_TAPS_L2 (1 input evict_last, 2 TMA-stored output evict_first) x LCNN_TAPS_TMA
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/tl
: > gpurun_out/tl/ab.jsonl
for r in 1 2; do for cfg in "0 1" "1 1" "3 1" "3 2" "1 0"; do
  set -- $cfg
  echo "{\"l2\": $1, \"tma\": $2}" >> gpurun_out/tl/ab.jsonl
  LCNN_TAPS_L2=$1 LCNN_TAPS_TMA=$2 timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/tl/ab.jsonl 2>> gpurun_out/tl/err.log
done; done
LCNN_TAPS_L2=3 LCNN_TAPS_TMA=2 timeout 600 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "conv_chwn or sync" > gpurun_out/tl/test.log 2>&1; echo rc=$? >> gpurun_out/tl/test.log
echo done
