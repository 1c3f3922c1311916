# quick A/B of single-op bench lines: bash scripts/ab_quick.sh TAG [workloads...]
set -u
cd ${GRAFT_REPO_ROOT:-.}
tag=$1; shift
for wl in "$@"; do
  if [ $wl = default ]; then a=""; else a="--workload $wl"; fi
  timeout 200 python bench.py $a --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | sed "s/^/$tag /" >> gpurun_out/ab.txt
done
