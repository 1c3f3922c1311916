# A/B of the in-tree build against ab_old/*.so (a previous build), alternating
# runs on the same box: bash scripts/ab_libs.sh ROUNDS workload...
set -u
cd ${GRAFT_REPO_ROOT:-.}
L=paper_1610_03618_b200/lib
mkdir -p /tmp/ab_new && cp $L/*.so /tmp/ab_new/
rounds=$1; shift
: > gpurun_out/ab.txt
for r in $(seq 1 $rounds); do
  for v in old new; do
    if [ $v = old ]; then cp ab_old/*.so $L/; else cp /tmp/ab_new/*.so $L/; fi
    bash scripts/ab_quick.sh $v "$@"
  done
done
cp /tmp/ab_new/*.so $L/
