set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv_pool.py -x -q > gpurun_out/fuse_test.log 2>&1; echo "rc=$?" >> gpurun_out/fuse_test.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "alexnet" > gpurun_out/fuse_full.log 2>&1; echo "rc=$?" >> gpurun_out/fuse_full.log
: > gpurun_out/fuse_bench.jsonl
for f in 1 0; do
LCNN_FUSE_POOL=$f timeout 600 python bench.py --workload alexnet --steps 50 --no-cpu-baseline >> gpurun_out/fuse_bench.jsonl 2>> gpurun_out/fuse_bench.err
done
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/fuse_launches.csv python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
