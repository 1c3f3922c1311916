set -u
cd $GRAFT_REPO_ROOT
run() { tag=$1
  for wl in alexnet alexnet vgg16; do timeout 200 python bench.py --workload $wl --steps 30 --no-cpu-baseline --no-e2e | sed "s/^/$tag /" >> gpurun_out/cs_ab.txt; done
  for wl in pl5 default; do if [ $wl = default ]; then a=""; else a="--workload $wl"; fi; timeout 200 python bench.py $a --steps 20 --no-cpu-baseline --no-e2e | sed "s/^/$tag /" >> gpurun_out/cs_ab.txt; done
}
: > gpurun_out/cs_ab.txt
run cs1
make -B -j16 EXTRA_NVFLAGS=-DLCNN_CS_STORES=0 > gpurun_out/cs_build.txt 2>&1
run cs0
