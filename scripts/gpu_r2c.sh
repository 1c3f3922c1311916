#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/bench2.jsonl
for wl in alexnet vgg16 alexnet_mixed; do
  timeout 600 python bench.py --workload $wl --steps 50 --no-cpu-baseline >> gpurun_out/bench2.jsonl 2>> gpurun_out/bench2.err
done
LCNN_SHAREPOOL_STORE=tma timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e >> gpurun_out/bench2.jsonl 2>> gpurun_out/bench2.err
timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline --no-e2e --no-graph >> gpurun_out/bench2.jsonl 2>> gpurun_out/bench2.err
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 200 --csv --log-file gpurun_out/launches_alexnet_direct.csv \
  python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
