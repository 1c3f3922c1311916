#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transform.py "tests/test_gpu_fullsize.py::test_bench_transform_workloads_bit_exact" tests/test_gpu_softmax.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
# fc split-K A/B on AlexNet (per-entry spans) + its parity under the knob
for v in 1 2; do
  LCNN_FC_SPLITK=$v timeout 600 python bench.py --workload alexnet --steps 50 --no-e2e --no-cpu-baseline >> gpurun_out/fc_splitk_ab.jsonl 2>/dev/null
done
LCNN_FC_SPLITK=2 timeout 600 python -m pytest tests/test_gpu_conv_gemm.py -q -x -k "fc or gemm" >> gpurun_out/pytest_gpu.log 2>&1; echo "splitk2 pytest rc=$?" >> gpurun_out/pytest_gpu.log
LCNN_FC_SPLITK=2 timeout 600 python -m pytest "tests/test_gpu_fullsize.py::test_alexnet_forward_fullsize_vs_reference" -q -x >> gpurun_out/pytest_gpu.log 2>&1; echo "splitk2 alexnet rc=$?" >> gpurun_out/pytest_gpu.log
bash scripts/bench_sweeps.sh
echo done
