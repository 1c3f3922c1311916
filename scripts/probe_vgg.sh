#!/bin/bash
# PROFILING build: LCNN_TC_PROBE 0 / 1 (no MMA) / 2 (no epilogue stores) / 3 (loads only) on the
# VGG TAPS layers (conv1_2 row pairs, conv2_1, conv2_2); PROBES="0 8 3 11" adds bit 8 (TAPS:
# filter slices loaded for the first tile only)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/pv
touch paper_1610_03618_b200/csrc/*.cu; make PROFILING=1 -j16 > gpurun_out/pv/build.log 2>&1
: > gpurun_out/pv/probe.txt
for p in ${PROBES:-0 1 2 3}; do
  echo "probe $p $(LCNN_TC_PROBE=$p timeout 300 python scripts/perf_dense.py ${LAYERS:-vgg1_2_chwn vgg2_1_chwn vgg2_2_chwn} 2>&1 | tail -1)" >> gpurun_out/pv/probe.txt
done
echo done
