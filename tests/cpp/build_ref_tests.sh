#!/bin/bash
# Compile the reference's OWN unit tests and acceptance gate, unmodified, from
# where they lie (/root/reference/proj/tests), against the B200 lcnn library
# (paper_1610_03618_b200/lib/liblcnn.so + host/include) and the doctest shim.
# The binaries land in build/reftests/ (git-ignored) and travel to the GPU box
# with the snapshot; tests/test_gpu_reftests.py runs them there.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${LCNN_REFERENCE_DIR:-/root/reference/proj}
OUT=$ROOT/build/reftests
if [ ! -d "$REF/tests" ]; then echo "no reference tests at $REF"; exit 0; fi
mkdir -p "$OUT"
CXXFLAGS="-std=c++20 -O2 -I$ROOT/tests/cpp/doctest_shim -I$ROOT/paper_1610_03618_b200/host/include -I$ROOT/include"
LIBS="-L$ROOT/paper_1610_03618_b200/lib -llcnn -llcnn_cuda -Wl,-rpath,$ROOT/paper_1610_03618_b200/lib -Wl,-rpath,\$ORIGIN/../../paper_1610_03618_b200/lib"
g++ $CXXFLAGS -c "$REF/tests/doctest_main.cpp" -o "$OUT/doctest_main.o"
for t in test_tensor test_layout test_pool test_softmax test_select test_conv test_net test_bench; do
  g++ $CXXFLAGS "$REF/tests/$t.cpp" "$OUT/doctest_main.o" -o "$OUT/$t" $LIBS &
done
g++ $CXXFLAGS "$REF/tests/acceptance.cpp" -o "$OUT/acceptance" $LIBS &
wait
ls "$OUT"
