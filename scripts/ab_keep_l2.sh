#!/bin/bash
# conv2 output stores with an L2 evict_last hint (LCNN_KEEP_L2=1) so pool2 reads it from L2
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/kl
: > gpurun_out/kl/ab.jsonl
for r in 1 2 3; do for k in 0 1 2; do
  echo "{\"keep\": $k}" >> gpurun_out/kl/ab.jsonl
  LCNN_KEEP_L2=$k timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e >> gpurun_out/kl/ab.jsonl 2>> gpurun_out/kl/err.log
done; done
LCNN_KEEP_L2=2 timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "alexnet_forward" > gpurun_out/kl/test.log 2>&1; echo rc=$? >> gpurun_out/kl/test.log
echo done
