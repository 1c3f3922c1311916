#!/bin/bash
# fc layers prefetch the next fc's packed weights into L2 as they drain (LCNN_FC_NEXT_PREFETCH)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/fn
timeout 600 python -m pytest tests/test_gpu_conv_gemm.py tests/test_gpu_fullsize.py -x -q -k "fc_packed or alexnet_forward" > gpurun_out/fn/test.log 2>&1; echo rc=$? >> gpurun_out/fn/test.log
: > gpurun_out/fn/ab.jsonl
for r in 1 2 3; do for k in 1 0; do
  echo "{\"next\": $k}" >> gpurun_out/fn/ab.jsonl
  LCNN_FC_NEXT_PREFETCH=$k timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e >> gpurun_out/fn/ab.jsonl 2>> gpurun_out/fn/err.log
done; done
echo done
