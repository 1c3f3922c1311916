#!/bin/bash
# Softmax 4096x1000 (BASELINE config 2): kernel variants against the
# same-size copy ceiling, and the rows sweep.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sm
: > gpurun_out/sm/bench.jsonl
for cfg in base "LCNN_SOFTMAX_PF=1" base "LCNN_SOFTMAX_PF=1"; do
  envs=""; [ "$cfg" != base ] && envs="$cfg"
  env $envs timeout 300 python bench.py --workload softmax --steps 200 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['ab']='$cfg'; print(json.dumps(d))" >> gpurun_out/sm/bench.jsonl 2>> gpurun_out/sm/err.log
done
for wl in transform softmax_64k; do
  timeout 300 python bench.py --workload $wl --steps 50 --no-cpu-baseline --no-e2e >> gpurun_out/sm/bench.jsonl 2>> gpurun_out/sm/err.log
done
echo done
