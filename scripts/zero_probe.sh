#!/bin/bash
# What the stream-K zeroing launches cost: PROFILING build, AlexNet forward
# and the cold fc probe with and without LCNN_SKIP_ZERO (wrong sums; timing only).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/zp
touch paper_1610_03618_b200/csrc/*.cu; make PROFILING=1 -j16 > gpurun_out/zp/build.log 2>&1
: > gpurun_out/zp/out.jsonl
for z in 0 1 0 1; do
  LCNN_SKIP_ZERO=$z timeout 300 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e \
   | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'skip':$z,'v':d['value'],'ms':d['ms_per_step']}))" >> gpurun_out/zp/out.jsonl 2>> gpurun_out/zp/err.log
  LCNN_SKIP_ZERO=$z timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/zp/out.jsonl 2>> gpurun_out/zp/err.log
done
echo done
