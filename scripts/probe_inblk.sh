cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for p in 0 1; do
  echo "inblk $p $(LCNN_TAPS_INBLK=$p timeout 300 python scripts/perf_dense.py vgg1_2_chwn vgg2_1_chwn vgg2_2_chwn 2>&1 | tail -1)" >> gpurun_out/inblk.txt
done; done
