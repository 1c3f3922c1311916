#!/bin/bash
# ncu evidence for round 2: launch lists (cold-cache per-launch times) and
# --set full captures of the dominant kernels, restricted to bench.py's timed
# region (NVTX range "timed"; the tuner's and warm-up launches are outside).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NV="--nvtx --nvtx-include timed/"
for WHAT in ${@:-softmax vgg}; do
case $WHAT in
  softmax)
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:softmax -c 1 \
      -o gpurun_out/r02_softmax -f python bench.py --workload softmax --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_softmax.log 2>&1
    timeout 600 ncu $NV --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/r02_softmax_launches.csv python bench.py --workload softmax --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
    ;;
  vgg)
    timeout 600 ncu $NV --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/r02_launches_vgg.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:pool -c 1 \
      -o gpurun_out/r02_pool_vgg1 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pool.log 2>&1
    ;;
esac
done
echo done
