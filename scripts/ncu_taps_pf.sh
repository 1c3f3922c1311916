#!/bin/bash
# ncu of the VGG conv1_2 TAPS kernel with and without the whole-row L2 prefetch (LCNN_TAPS_PF)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/npf
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum
for p in 0 2; do
  LCNN_TAPS_PF=$p timeout 600 ncu --metrics $M --clock-control none -k regex:tc_conv_taps -c 2 --csv \
    python scripts/perf_dense.py vgg1_2_chwn > gpurun_out/npf/pf$p.csv 2>&1
done
echo done
