#!/bin/bash
# TAPS / TAPS-N in-kernel zeroing: parity + VGG A/B; small-N transform sweep
# with the graph-timed dominant kernel.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/z
timeout 900 python -m pytest tests/test_gpu_conv_gemm.py tests/test_gpu_transform.py -x -q > gpurun_out/z/test.log 2>&1; echo "rc=$?" >> gpurun_out/z/test.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "vgg16 or transform" > gpurun_out/z/test_full.log 2>&1; echo "rc=$?" >> gpurun_out/z/test_full.log
: > gpurun_out/z/ab.jsonl
for r in 1 2; do for k in 1 0; do
  echo "{\"kz\": $k}" >> gpurun_out/z/ab.jsonl
  LCNN_KERNEL_ZERO=$k timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/z/ab.jsonl 2>> gpurun_out/z/err.log
done; done
: > gpurun_out/z/tsmall.jsonl
for n in 1 2 4 8 16 32 64 128 256; do
  timeout 300 python bench.py --workload transform_$n --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/z/tsmall.jsonl 2>> gpurun_out/z/err.log
  timeout 300 python bench.py --workload transform_nchw_$n --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/z/tsmall.jsonl 2>> gpurun_out/z/err.log
done
echo done
