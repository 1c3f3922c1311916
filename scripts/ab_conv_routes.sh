#!/bin/bash
# A/B of conv routing knobs on the AlexNet forward: per-launch times (ncu
# launch list, cold) and the bench step for each setting.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ab
: > gpurun_out/ab/bench.jsonl
for cfg in "base" "LCNN_CONV_PAIR=2" "LCNN_CONV_PAIR=2 LCNN_STREAMK=0" "LCNN_STREAMK=0" ${EXTRA_CFGS:-}; do
  tag=$(echo "$cfg" | tr ' =' '_-')
  envs=""; [ "$cfg" != base ] && envs="$cfg"
  env $envs timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e \
     | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['ab']='$cfg'; print(json.dumps(d))" >> gpurun_out/ab/bench.jsonl 2>> gpurun_out/ab/err.log
  env $envs timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none -c 200 --csv --log-file gpurun_out/ab/launches_$tag.csv \
     python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
echo done
