set -u
cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out/ncu_conv
N="ncu --set full --clock-control none --import-source on -f -k regex:tc_gemm_persistent -s 3 -c 1"
for c in conv1_chwn conv2_chwn conv4_chwn; do
  timeout 300 $N -o gpurun_out/ncu_conv/$c python scripts/perf_dense.py $c > /dev/null 2>&1
  ncu -i gpurun_out/ncu_conv/$c.ncu-rep --page details --csv > gpurun_out/ncu_conv/${c}_details.csv 2>/dev/null
  ncu -i gpurun_out/ncu_conv/$c.ncu-rep --page raw --csv > gpurun_out/ncu_conv/${c}_raw.csv 2>/dev/null
done
ls -la gpurun_out/ncu_conv
