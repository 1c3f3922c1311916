#!/bin/bash
# One gpurun session: parity tests, smoke, bench lines, ncu launch list and
# --set full captures of the dominant kernels.  Outputs land in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
STAGE=${1:-all}
if [[ $STAGE == all || $STAGE == test ]]; then
  timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [[ $STAGE == all || $STAGE == bench ]]; then
  : > gpurun_out/bench.jsonl
  timeout 600 python bench.py >> gpurun_out/bench.jsonl 2> gpurun_out/bench.err
  for wl in vgg_pools_nchw pl5 pl5_nchw softmax softmax5 softmax_64k transform alexnet vgg16; do
    timeout 300 python bench.py --workload $wl --steps 50 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
  done
  timeout 300 python bench.py --impl reference --steps 3 --warmup 3 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
  timeout 300 python bench.py --workload alexnet --impl reference --steps 2 --warmup 1 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
fi
if [[ $STAGE == all || $STAGE == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_vgg.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_chwn -s 5 -c 1 \
    -o gpurun_out/prof_pool_vgg1 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pool.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_chwn -s 3 -c 1 \
    -o gpurun_out/prof_pool_pl5 -f python bench.py --workload pl5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_nchw -s 3 -c 1 \
    -o gpurun_out/prof_pool_pl5nchw -f python bench.py --workload pl5_nchw --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:transpose -s 27 -c 1 \
    -o gpurun_out/prof_transform -f python bench.py --workload transform --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmax -s 3 -c 1 \
    -o gpurun_out/prof_softmax -f python bench.py --workload softmax --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
fi
echo done
