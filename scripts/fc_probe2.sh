#!/bin/bash
# fc activation-traffic probe (PROFILING build): LCNN_TC_PROBE bit 4 skips the
# activation (A) loads of the packed fc, so 4 / 6 / 7 split how much of the
# fc time the per-n-tile activation re-reads cost (0 = shipped kernel,
# 3 = loads only, 7 = weight loads only).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/fc
: > gpurun_out/fc/probe2.jsonl
touch paper_1610_03618_b200/csrc/*.cu; make PROFILING=1 -j16 > gpurun_out/fc/build.log 2>&1
for p in ${PROBES:-0 4 6 3 7}; do LCNN_TC_PROBE=$p timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/fc/probe2.jsonl 2>> gpurun_out/fc/err.log; done
echo done
