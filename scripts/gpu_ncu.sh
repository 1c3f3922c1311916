#!/bin/bash
# ncu --set full captures of the current hot kernels (one launch each) and the
# launch lists of the default bench, into gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --no-graph"
N="ncu --set full --clock-control none --import-source on -f"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_vgg.csv $B --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:pool_chwn -s 5 -c 1 -o gpurun_out/prof_vgg_pool1 $B --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:pool_nchw -s 5 -c 1 -o gpurun_out/prof_vgg_pool1_nchw $B --workload vgg_pools_nchw --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:pool_chwn -s 3 -c 1 -o gpurun_out/prof_pl5 $B --workload pl5 --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:pool_nchw -s 3 -c 1 -o gpurun_out/prof_pl5_nchw $B --workload pl5_nchw --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:softmax -s 3 -c 1 -o gpurun_out/prof_softmax $B --workload softmax --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:softmax -s 3 -c 1 -o gpurun_out/prof_softmax_64k $B --workload softmax_64k --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:transpose -s 27 -c 1 -o gpurun_out/prof_transform $B --workload transform --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $N -k regex:tc_gemm -s 8 -c 2 -o gpurun_out/prof_alexnet_conv $B --workload alexnet --steps 1 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
# summarise on the box; keep the returned payload small
python scripts/ncu_summary.py launches gpurun_out/launches_vgg.csv gpurun_out/launches_vgg.md
python scripts/ncu_summary.py full gpurun_out/ncu_full.json gpurun_out/prof_*.ncu-rep
for f in gpurun_out/prof_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page details --csv > gpurun_out/${b}_details.csv 2>/dev/null
done
mkdir -p gpurun_out/reps
for f in gpurun_out/prof_*.ncu-rep; do
  s=$(stat -c %s $f); if [ $s -lt 4000000 ]; then mv $f gpurun_out/reps/; else rm -f $f; fi
done
du -sh gpurun_out
