#!/bin/bash
# TAPS with two accumulators (row pairs for C_o > 64; VGG conv2_1, conv2_2 (+ pool2 fused))
# against one output row per tile (LCNN_TAPS_ACC2=0): parity, then alternating VGG-16 forwards
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/a2
timeout 1500 python -m pytest tests/test_gpu_conv_gemm.py tests/test_gpu_conv_pool.py tests/test_gpu_fullsize.py -x -q > gpurun_out/a2/test.log 2>&1; echo rc=$? >> gpurun_out/a2/test.log
for k in 1 0; do
  echo "acc2 $k $(LCNN_TAPS_ACC2=$k timeout 300 python scripts/perf_dense.py vgg2_1_chwn vgg2_2_chwn 2>&1 | tail -1)" >> gpurun_out/a2/dense.txt
done
: > gpurun_out/a2/ab.jsonl
for r in 1 2; do for k in 1 0; do
  echo "{\"acc2\": $k}" >> gpurun_out/a2/ab.jsonl
  LCNN_TAPS_ACC2=$k timeout 600 python bench.py --workload vgg16 --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/a2/ab.jsonl 2>> gpurun_out/a2/err.log
done; done
echo done
