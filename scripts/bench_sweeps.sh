#!/bin/bash
# Builder-kept bench lines for BASELINE configs 1, 2, 3 and 5 (the driver runs
# only the default config 4): softmax fused vs five-kernel over N = 128..4096
# (+ the 65536-row asymptote), the transform sweep N in {32,64,128,256} in both
# directions, PL5 in both layouts, AlexNet (selector / mixed layouts), VGG-16.
# One JSON line per run into gpurun_out/sweeps.jsonl.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/sweeps.jsonl
: > $OUT
run() { timeout 900 python bench.py "$@" >> $OUT 2>> gpurun_out/sweeps.err; }
for what in ${@:-softmax transform transform_small pl5 nets}; do
case $what in
  softmax)
    for n in 128 256 512 1024 2048 4096; do
      run --workload softmax_$n --steps 200 --ref-sample-gb 0
      run --workload softmax5_$n --steps 200 --no-cpu-baseline
    done
    run --workload softmax_64k --steps 50
    ;;
  transform)
    for n in 32 64 128 256; do
      run --workload transform_$n --steps 10
      run --workload transform_nchw_$n --steps 10
    done
    ;;
  transform_small)
    for n in 1 2 4 8 16; do
      run --workload transform_$n --steps 20 --no-cpu-baseline
      run --workload transform_nchw_$n --steps 20 --no-cpu-baseline
    done
    ;;
  pl5)
    run --workload pl5 --steps 200
    run --workload pl5_nchw --steps 200
    ;;
  nets)
    run --workload alexnet --steps 50
    run --workload alexnet_mixed --steps 50
    run --workload vgg16 --steps 10
    ;;
esac
done
echo done
