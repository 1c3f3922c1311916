#!/bin/bash
# ncu --set full of AlexNet conv3/conv4/conv5 (CHWN, TF32) one CTA per tile
# (RowsOut, the shipped route) and on the CTA pair (LCNN_CONV_PAIR=2).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/c345
for c in conv3_chwn conv4_chwn conv5_chwn; do
  timeout 300 ncu --set full --clock-control none --import-source on -f -k regex:tc_gemm_persistent -s 3 -c 1 \
    -o gpurun_out/c345/${c}_single python scripts/perf_dense.py $c > /dev/null 2>&1
  LCNN_CONV_PAIR=2 timeout 300 ncu --set full --clock-control none --import-source on -f -k regex:tc_gemm_pair -s 3 -c 1 \
    -o gpurun_out/c345/${c}_pair python scripts/perf_dense.py $c > /dev/null 2>&1
done
for r in gpurun_out/c345/*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}.details.csv" 2>/dev/null
  rm -f "$r"
done
python scripts/perf_dense.py conv3_chwn conv4_chwn conv5_chwn > gpurun_out/c345/perf_single.json 2>&1
LCNN_CONV_PAIR=2 python scripts/perf_dense.py conv3_chwn conv4_chwn conv5_chwn > gpurun_out/c345/perf_pair.json 2>&1
echo done
