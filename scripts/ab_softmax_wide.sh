#!/bin/bash
# wide-row softmax occupancy bounds (LCNN_SM_WIDE_MINB=1 disables them) across widths
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sw
timeout 300 python -m pytest tests/test_gpu_softmax.py -x -q > gpurun_out/sw/test.log 2>&1; echo rc=$? >> gpurun_out/sw/test.log
: > gpurun_out/sw/b.jsonl
for c in 4096 8192 10000 12288 16384; do for k in 0 1; do
  echo "{\"minb1\": $k, \"cols\": $c}" >> gpurun_out/sw/b.jsonl
  LCNN_SM_WIDE_MINB=$k timeout 600 python bench.py --workload softmax_c$c --steps 30 --no-cpu-baseline --no-e2e >> gpurun_out/sw/b.jsonl 2>> gpurun_out/sw/err.log
done; done
echo done
