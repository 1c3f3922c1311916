#!/bin/bash
# ROW row pairs (VGG conv1_1): parity + VGG A/B; transform small-N sweep with
# graph-timed steps; fc6 ncu capture.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/rows2
timeout 900 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "conv" > gpurun_out/rows2/test.log 2>&1; echo "rc=$?" >> gpurun_out/rows2/test.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "conv_routes or vgg16" > gpurun_out/rows2/test_full.log 2>&1; echo "rc=$?" >> gpurun_out/rows2/test_full.log
: > gpurun_out/rows2/ab.jsonl
for r in 1 2; do for k in 1 0; do
  echo "{\"row2\": $k}" >> gpurun_out/rows2/ab.jsonl
  LCNN_CONV_ROW2=$k timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/rows2/ab.jsonl 2>> gpurun_out/rows2/err.log
done; done
: > gpurun_out/rows2/tsmall.jsonl
for n in 1 2 4 8 16 32; do
  timeout 300 python bench.py --workload transform_$n --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/rows2/tsmall.jsonl 2>> gpurun_out/rows2/err.log
  timeout 300 python bench.py --workload transform_nchw_$n --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/rows2/tsmall.jsonl 2>> gpurun_out/rows2/err.log
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/rows2/tsmall.jsonl 2>> gpurun_out/rows2/err.log
bash scripts/gpu_ncu_r2.sh nets
echo done
