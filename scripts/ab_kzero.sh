#!/bin/bash
# A/B on one box: stream-K zeroing in-kernel (sync words) vs zero2d launches.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/kz
: > gpurun_out/kz/ab.jsonl
for r in 1 2 3; do
for kz in 1 0; do
  echo "{\"kz\": $kz}" >> gpurun_out/kz/ab.jsonl
  LCNN_KERNEL_ZERO=$kz timeout 300 python bench.py --workload ${WL:-alexnet} --steps 100 --no-cpu-baseline --no-e2e >> gpurun_out/kz/ab.jsonl 2>> gpurun_out/kz/err.log
done
done
echo done
