#!/bin/bash
# Round-2 second session: full GPU suite + smoke, sanitizers over the new
# fused kernel, default bench + reference arm + AlexNet/VGG/softmax lines, and
# the ncu evidence of the fused AlexNet forward.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash scripts/sanitize_r2.sh > /dev/null 2>&1
: > gpurun_out/bench.jsonl
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 >> gpurun_out/bench.jsonl 2> gpurun_out/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
for wl in alexnet vgg16 softmax alexnet_mixed; do
  timeout 600 python bench.py --workload $wl --steps 50 >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
done
O=gpurun_out/ncu_fused; mkdir -p $O
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 200 --csv --log-file $O/launches_alexnet.csv \
  python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on \
  -k regex:tc_gemm_persistent -c 1 -o $O/conv1pool1 -f \
  python bench.py --workload alexnet --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/conv1pool1.ncu-rep --page raw --csv > $O/conv1pool1_raw.csv 2>/dev/null
ncu -i $O/conv1pool1.ncu-rep --page details --csv > $O/conv1pool1_details.csv 2>/dev/null
ncu -i $O/conv1pool1.ncu-rep --page source --csv > $O/conv1pool1_source.csv 2>/dev/null
rm -f $O/*.ncu-rep
echo done
