#!/bin/bash
# stream-K tail threshold A/B (LCNN_SK_FULL_PCT) now that the zeroing is in-kernel
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sk
: > gpurun_out/sk/ab.jsonl
for r in 1 2; do for k in 60 80 101; do
  echo "{\"pct\": $k}" >> gpurun_out/sk/ab.jsonl
  LCNN_SK_FULL_PCT=$k timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e >> gpurun_out/sk/ab.jsonl 2>> gpurun_out/sk/err.log
done; done
echo done
