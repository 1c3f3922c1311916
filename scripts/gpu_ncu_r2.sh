#!/bin/bash
# ncu evidence for round 2: launch lists (cold-cache per-launch times) and
# --set full captures of the dominant kernels, restricted to bench.py's timed
# region (NVTX range "timed"; the tuner's and warm-up launches are outside).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NV="--nvtx --nvtx-include timed/"
LM="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
B="--no-e2e --no-cpu-baseline"
for WHAT in ${@:-vgg softmax pl5 transform alexnet}; do
case $WHAT in
  vgg)
    timeout 600 ncu $NV --metrics $LM --clock-control none -c 400 --csv \
      --log-file gpurun_out/r02_launches_vgg.csv python bench.py --steps 2 --warmup 3 $B > /dev/null 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:pool -c 1 \
      -o gpurun_out/r02_pool_vgg1 -f python bench.py --steps 1 --warmup 3 $B > gpurun_out/ncu_pool.log 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:pool -c 1 \
      -o gpurun_out/r02_pool_vgg1_nchw -f python bench.py --workload vgg_pools_nchw --steps 1 --warmup 3 $B > /dev/null 2>&1
    ;;
  softmax)
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:softmax -c 1 \
      -o gpurun_out/r02_softmax -f python bench.py --workload softmax --steps 2 --warmup 3 $B --no-graph > gpurun_out/ncu_softmax.log 2>&1
    timeout 600 ncu $NV --metrics $LM --clock-control none -c 60 --csv \
      --log-file gpurun_out/r02_softmax_launches.csv python bench.py --workload softmax --steps 20 --warmup 3 $B --no-graph > /dev/null 2>&1
    ;;
  pl5)
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:pool -c 1 \
      -o gpurun_out/r02_pool_pl5 -f python bench.py --workload pl5 --steps 2 --warmup 3 $B --no-graph > /dev/null 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:pool -c 1 \
      -o gpurun_out/r02_pool_pl5_nchw -f python bench.py --workload pl5_nchw --steps 2 --warmup 3 $B --no-graph > /dev/null 2>&1
    ;;
  transform)
    timeout 600 ncu $NV --metrics $LM --clock-control none -c 100 --csv \
      --log-file gpurun_out/r02_launches_transform.csv python bench.py --workload transform --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:transpose -s 9 -c 1 \
      -o gpurun_out/r02_transform -f python bench.py --workload transform --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:transpose_small -c 1 \
      -o gpurun_out/r02_transform_small -f python bench.py --workload transform_nchw_8 --steps 1 --warmup 3 $B > /dev/null 2>&1
    ;;
  alexnet)
    timeout 600 ncu $NV --metrics $LM --clock-control none -c 200 --csv \
      --log-file gpurun_out/r02_launches_alexnet.csv python bench.py --workload alexnet --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 600 ncu $NV --metrics $LM --clock-control none -c 200 --csv \
      --log-file gpurun_out/r02_launches_alexnet_mixed.csv python bench.py --workload alexnet_mixed --steps 1 --warmup 3 $B > /dev/null 2>&1
    ;;
  nets)
    timeout 900 ncu $NV --metrics $LM --clock-control none -c 200 --csv \
      --log-file gpurun_out/r02_launches_vgg16.csv python bench.py --workload vgg16 --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 600 ncu $NV --set full --clock-control none --import-source on -k regex:tc_gemm_persistent -s 4 -c 1 \
      -o gpurun_out/r02_fc6 -f python bench.py --workload alexnet --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 900 ncu $NV --set full --clock-control none --import-source on -k regex:tc_conv_taps_kernel -c 1 \
      -o gpurun_out/r02_vgg_conv1_2 -f python bench.py --workload vgg16 --steps 1 --warmup 3 $B > /dev/null 2>&1
    ;;
  vggfused)  # VGG-16 with conv1_2 -> pool1 fused (TAPS row-pair epilogue pool)
    timeout 900 ncu $NV --metrics $LM --clock-control none -c 200 --csv \
      --log-file gpurun_out/r02_launches_vgg16.csv python bench.py --workload vgg16 --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 900 ncu $NV --set full --clock-control none --import-source on -k regex:tc_conv_taps_kernel -c 1 \
      -o gpurun_out/r02_vgg_conv1_2_pool -f python bench.py --workload vgg16 --steps 1 --warmup 3 $B > /dev/null 2>&1
    timeout 600 ncu $NV --metrics $LM --clock-control none -c 200 --csv \
      --log-file gpurun_out/r02_launches_alexnet.csv python bench.py --workload alexnet --steps 1 --warmup 3 $B > /dev/null 2>&1
    ;;
esac
done
# keep gpurun_out small (the pull limit is 64 MiB): text exports of every
# report, the .ncu-rep files themselves only with KEEP_REP=1
for r in gpurun_out/*.ncu-rep; do
  [ -e "$r" ] || continue
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}.details.csv" 2>/dev/null
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page source --csv > "${r%.ncu-rep}.source.csv" 2>/dev/null
  [ "${KEEP_REP:-0}" = 1 ] || rm -f "$r"
done
du -sh gpurun_out
echo done
