#!/bin/bash
# ncu --set full of the AlexNet fc layers (fc6 FcLoader<1>, fc7 FcLoader<0>) in
# bench.py's timed region; raw metrics exported as CSV.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/ncu_fc; mkdir -p $O
B="python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on \
  -k regex:tc_gemm_persistent -s 4 -c 2 -o $O/fc -f $B > $O/ncu.log 2>&1
ncu -i $O/fc.ncu-rep --page raw --csv > $O/fc_raw.csv 2>/dev/null
ncu -i $O/fc.ncu-rep --page details --csv > $O/fc_details.csv 2>/dev/null
rm -f $O/fc.ncu-rep
echo done
