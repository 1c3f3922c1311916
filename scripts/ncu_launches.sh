#!/bin/bash
# ncu launch list (duration + DRAM bytes per kernel) of one workload:
#   bash scripts/ncu_launches.sh <workload> <out.csv> [count]
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c ${3:-60} --csv --log-file gpurun_out/$2 \
  python bench.py --workload $1 --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/$2 gpurun_out/${2%.csv}.md
