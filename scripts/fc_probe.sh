#!/bin/bash
# fc probes: shipped build (stream-K / split-K), then a PROFILING build with
# LCNN_TC_PROBE 1 (no MMA) / 2 (no epilogue stores) / 3 (loads only).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/fc
: > gpurun_out/fc/probe.jsonl
for sk in ${SKS:-}; do LCNN_FC_SPLITK=$sk timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/fc/probe.jsonl 2>> gpurun_out/fc/err.log; done
touch paper_1610_03618_b200/csrc/*.cu; make PROFILING=1 -j16 > gpurun_out/fc/build.log 2>&1
for p in 0 1 2 3; do LCNN_TC_PROBE=$p timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/fc/probe.jsonl 2>> gpurun_out/fc/err.log; done
echo done
