#!/bin/bash
# PROFILING build: conv3/4/5 single-CTA vs CTA pair, LCNN_TC_PROBE 0 / 1 (no MMA) / 2 (no stores) / 3 (loads only)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/p345
touch paper_1610_03618_b200/csrc/*.cu; make PROFILING=1 -j16 > gpurun_out/p345/build.log 2>&1
: > gpurun_out/p345/probe.txt
for pair in 0 2; do for p in 0 1 2 3; do
  echo "pair $pair probe $p $(LCNN_CONV_PAIR=$pair LCNN_TC_PROBE=$p timeout 300 python scripts/perf_dense.py conv2_chwn conv3_chwn conv4_chwn conv5_chwn 2>&1 | tail -1)" >> gpurun_out/p345/probe.txt
done; done
echo done
