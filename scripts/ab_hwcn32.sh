#!/bin/bash
# Blocked [N/32][H][W][C][32] activation between VGG conv1_1 and conv1_2 + pool1:
# parity (pytest), then the VGG-16 forward with it on / off (LCNN_NET_HWCN32)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/hwcn32
timeout 900 python -m pytest tests -x -q -m gpu -k "hwcn32 or taps or vgg or conv_routes or net" \
  > gpurun_out/hwcn32/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hwcn32/pytest.log
: > gpurun_out/hwcn32/ab.jsonl
for r in 1 2; do for p in 1 0; do
  echo "{\"hwcn32\": $p}" >> gpurun_out/hwcn32/ab.jsonl
  LCNN_NET_HWCN32=$p timeout 600 python bench.py --workload vgg16 --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/hwcn32/ab.jsonl 2>> gpurun_out/hwcn32/err.log
done; done
echo done
