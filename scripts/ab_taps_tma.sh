#!/bin/bash
# TAPS TMA-store epilogue A/B on VGG-16 (LCNN_TAPS_TMA 0 off / 1 row pairs / 2 all) + parity
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/tt
LCNN_TAPS_TMA=2 timeout 600 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "conv_chwn or sync" > gpurun_out/tt/test.log 2>&1; echo rc=$? >> gpurun_out/tt/test.log
LCNN_TAPS_TMA=2 timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "conv_routes or vgg16" >> gpurun_out/tt/test.log 2>&1; echo rc=$? >> gpurun_out/tt/test.log
: > gpurun_out/tt/ab.jsonl
for r in 1 2; do for k in 0 1 2; do
  echo "{\"tma\": $k}" >> gpurun_out/tt/ab.jsonl
  LCNN_TAPS_TMA=$k timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/tt/ab.jsonl 2>> gpurun_out/tt/err.log
done; done
echo done
