#!/bin/bash
# ncu of the whole AlexNet forward: the launch list of one forward and --set
# full captures of conv1 (SHARE), conv2 (CTA pair), conv4, fc6 and fc8 (tcgen05
# kernel launches 0, 1, 3, 5, 7 of the warm-up forward), summarised on the box
# into gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ncu_alexnet
O=gpurun_out/ncu_alexnet
B="python bench.py --workload alexnet --no-e2e --no-cpu-baseline --steps 1 --warmup 1"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 60 --csv --log-file $O/launches.csv $B > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on -f -k regex:tc_gemm -c 1"
for pair in conv1:0 conv2:1 conv4:3 fc6:5 fc8:7; do
  name=${pair%%:*}; s=${pair##*:}
  timeout 600 $N -s $s -o $O/$name $B > /dev/null 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
done
python scripts/ncu_summary.py full $O/full.json $O/*.ncu-rep
for f in $O/*.ncu-rep; do s=$(stat -c %s $f); [ $s -gt 8000000 ] && rm -f $f; done
du -sh $O
