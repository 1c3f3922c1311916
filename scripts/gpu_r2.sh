#!/bin/bash
# Round-2 GPU session: parity (pytest -m gpu), smoke, the default bench line,
# the reference arm, and the extra workloads.  Outputs land in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt
STAGE=${1:-all}
if [[ $STAGE == all || $STAGE == test ]]; then
  timeout 2400 python -m pytest tests -x -q -m gpu --durations=25 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [[ $STAGE == all || $STAGE == bench ]]; then
  : > gpurun_out/bench.jsonl
  timeout 600 python bench.py --impl reference --steps 20 --warmup 5 >> gpurun_out/bench.jsonl 2> gpurun_out/bench.err
  timeout 600 python bench.py --steps 20 --warmup 5 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
  for wl in ${WORKLOADS:-}; do
    timeout 600 python bench.py --workload $wl --steps 50 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
  done
fi
echo done
