#!/bin/bash
# A/B of the fused classifier variants (LCNN_SOFTMAX_POLY) on B200: parity
# under each variant, then bench lines for 4096x1000 and 65536x1000.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/softmax_ab.txt
: > $OUT
for poly in 0 4 2; do
  LCNN_SOFTMAX_POLY=$poly timeout 600 python -m pytest tests/test_gpu_softmax.py "tests/test_gpu_fullsize.py::test_bench_softmax_workloads" -q -x 2>&1 | tail -1 | sed "s/^/poly=$poly pytest: /" >> $OUT
  for rep in 1 2 3; do
    for wl in softmax softmax_2048 softmax_64k; do
      LCNN_SOFTMAX_POLY=$poly timeout 300 python bench.py --workload $wl --steps 200 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('poly=$poly', '$wl', d['value'], d['roofline']['avg_launch_ms'])" >> $OUT
    done
  done
done
echo done
