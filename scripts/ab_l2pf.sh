#!/bin/bash
# A/B of the fc-weight L2 warm-up budget on the AlexNet / VGG-16 forwards.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/l2pf
: > gpurun_out/l2pf/bench.jsonl
for rep in 1 2; do
for cfg in "LCNN_FC_L2_PREFETCH_MB=0" "LCNN_FC_L2_PREFETCH_MB=32" "LCNN_FC_L2_PREFETCH_MB=64" "LCNN_FC_L2_PREFETCH_MB=96" "LCNN_FC_L2_PREFETCH_MB=128" "LCNN_FC_L2_PREFETCH_MB=64 LCNN_FC_L2_KEEP=0"; do
  env $cfg timeout 300 python bench.py --workload ${WL:-alexnet} --steps 50 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$cfg','v':d['value'],'ms':d['ms_per_step'],'pe':d['roofline'].get('per_entry_us')}))" >> gpurun_out/l2pf/bench.jsonl 2>> gpurun_out/l2pf/err.log
done
done
echo done
