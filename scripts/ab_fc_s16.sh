#!/bin/bash
# fc8 cluster split-K with clusters of 16 (LCNN_FC_S16=1) vs 8
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/s16
LCNN_FC_S16=1 timeout 600 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "fc_packed" > gpurun_out/s16/test.log 2>&1; echo rc=$? >> gpurun_out/s16/test.log
: > gpurun_out/s16/ab.jsonl
for k in 0 1; do LCNN_FC_S16=$k timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/s16/ab.jsonl 2>> gpurun_out/s16/err.log; done
for r in 1 2 3; do for k in 0 1; do
  echo "{\"s16\": $k}" >> gpurun_out/s16/ab.jsonl
  LCNN_FC_S16=$k timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e >> gpurun_out/s16/ab.jsonl 2>> gpurun_out/s16/err.log
done; done
echo done
