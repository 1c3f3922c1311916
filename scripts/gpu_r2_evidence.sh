#!/bin/bash
# Round-2 evidence refresh: full GPU suite + smoke, sweeps, ncu (nets).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash scripts/gpu_r2.sh test
bash scripts/bench_sweeps.sh ${SWEEPS:-transform_small softmax pl5 nets}
bash scripts/gpu_ncu_r2.sh ${NCU_WHAT:-nets}
echo done
