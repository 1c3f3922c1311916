#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/eb
timeout 900 python -m pytest tests/test_gpu_conv_gemm.py tests/test_gpu_fullsize.py -q -m gpu -k "fc or alexnet or vgg" > gpurun_out/eb/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/eb/pytest.log
: > gpurun_out/eb/out.jsonl
for i in 1 2; do
timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/eb/out.jsonl 2>> gpurun_out/eb/err.log
timeout 300 python bench.py --workload alexnet --steps 100 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'v':d['value'],'ms':d['ms_per_step'],'t':d['timing']}))" >> gpurun_out/eb/out.jsonl 2>> gpurun_out/eb/err.log
done
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 200 --csv --log-file gpurun_out/eb/launches.csv \
  python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
echo done
