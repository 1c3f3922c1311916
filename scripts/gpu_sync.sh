#!/bin/bash
# In-kernel stream-K zeroing (sync words): parity, fc cold timing with / without
# sync words, AlexNet forward.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sync
timeout 900 python -m pytest tests/test_gpu_conv_gemm.py -x -q -k "sync or fc_packed or conv_chwn" > gpurun_out/sync/test.log 2>&1; echo "rc=$?" >> gpurun_out/sync/test.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_net.py -x -q > gpurun_out/sync/test_net.log 2>&1; echo "rc=$?" >> gpurun_out/sync/test_net.log
: > gpurun_out/sync/fc.jsonl
for sy in 0 1; do LCNN_FC_SYNC=$sy timeout 300 python scripts/perf_fc_cold.py >> gpurun_out/sync/fc.jsonl 2>> gpurun_out/sync/err.log; done
: > gpurun_out/sync/bench.jsonl
timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline >> gpurun_out/sync/bench.jsonl 2>> gpurun_out/sync/err.log
timeout 600 python bench.py --workload vgg16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/sync/bench.jsonl 2>> gpurun_out/sync/err.log
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/sync/launches.csv python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
