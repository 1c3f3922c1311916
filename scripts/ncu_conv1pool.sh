#!/bin/bash
# ncu --set full of the fused AlexNet conv1 + pool1 kernel (SharePoolOut) inside the forward
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/c1
timeout 600 ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:tc_gemm_persistent -c 1 \
  -o gpurun_out/c1/conv1pool -f python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
r=gpurun_out/c1/conv1pool.ncu-rep
ncu -i $r --page raw --csv > gpurun_out/c1/conv1pool.raw.csv 2>/dev/null
ncu -i $r --page details --csv > gpurun_out/c1/conv1pool.details.csv 2>/dev/null
ncu -i $r --page source --csv --print-source sass > gpurun_out/c1/conv1pool.sass.csv 2>/dev/null
ncu -i $r --page source --csv > gpurun_out/c1/conv1pool.source.csv 2>/dev/null
rm -f $r
echo done
