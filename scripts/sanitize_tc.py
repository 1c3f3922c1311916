"""Small tcgen05 routes under compute-sanitizer (memcheck / racecheck):
SHARE, ROW-on-M, CI channels-on-M (RowsOut), CTA pair (ColsOut), TAPS-N,
TAPS, the fused SHARE conv + max pool, and the packed fc, each once at a
small shape."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_conv_gemm as t  # noqa: E402
import test_gpu_conv_pool as tp  # noqa: E402
from paper_1610_03618_b200 import lcnn  # noqa: E402

d = torch.device("cuda:0")
cases = [(64, 3, 35, 35, 96, 11, 4, 0),      # SHARE
         (32, 3, 12, 12, 20, 3, 1, 1),       # ROW on M (narrow filters)
         (32, 64, 13, 13, 96, 3, 1, 1),      # CI
         (128, 32, 27, 27, 192, 3, 1, 1),    # CTA pair
         (64, 32, 30, 30, 96, 3, 1, 1),      # TAPS-N
         (128, 32, 92, 92, 64, 3, 1, 1)]     # TAPS
for c in cases:
    t._check_conv(d, *c, t.CHWN, lcnn.TF32)
# NCHW through the CHWN route (transpose, conv, transpose in the workspace)
for c in [(32, 64, 13, 13, 96, 3, 1, 1), (64, 3, 35, 35, 96, 11, 4, 0)]:
    t._check_conv(d, *c, t.NCHW, lcnn.TF32)
# SHARE conv with the 3x3/s2 and 2x2/s2 max pools fused into its epilogue
tp._run(d, (32, 3, 67, 71, 40, 11, 4, 2, 3, 2))
tp._run(d, (64, 3, 96, 96, 96, 11, 4, 0, 2, 2))
print("ok")
