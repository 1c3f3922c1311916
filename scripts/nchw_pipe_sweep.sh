# LCNN_NCHW_PIPE sweep (slot KB, ring slots, CTAs per SM) on the NCHW pool workloads
cd ${GRAFT_REPO_ROOT:-.}
: > gpurun_out/nchw_sweep.txt
for cfg in ${CFGS:-24,3,3 48,2,2}; do
  for wl in ${WLS:-pl5_nchw vgg_pools_nchw}; do
    v=$(LCNN_NCHW_PIPE=$cfg timeout 120 python bench.py --workload $wl --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])")
    echo "$cfg $wl $v" >> gpurun_out/nchw_sweep.txt
  done
done
