#!/bin/bash
# TAPS input rows prefetched into L2 (whole contiguous (c, h) rows) LCNN_TAPS_PF tile rows ahead
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/pf
: > gpurun_out/pf/dense.txt
for r in 1 2; do for p in 0 1 2 4 8; do
  echo "pf $p $(LCNN_TAPS_PF=$p timeout 300 python scripts/perf_dense.py vgg1_2_chwn vgg2_1_chwn vgg2_2_chwn 2>&1 | tail -1)" >> gpurun_out/pf/dense.txt
done; done
: > gpurun_out/pf/ab.jsonl
for r in 1 2; do for p in ${NETPF:-2 0}; do
  echo "{\"pf\": $p}" >> gpurun_out/pf/ab.jsonl
  LCNN_TAPS_PF=$p timeout 600 python bench.py --workload vgg16 --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/pf/ab.jsonl 2>> gpurun_out/pf/err.log
done; done
echo done
