"""Small tcgen05 routes under compute-sanitizer (memcheck / racecheck):
SHARE, ROW-on-M, CI channels-on-M (RowsOut), CTA pair (ColsOut), TAPS-N,
TAPS, the fused SHARE conv + max pool, the packed fc, ROW row pairs with
quad-chunk stores and TAPS row pairs with the fused 2x2 pool, each once at a
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
# round 2: stream-K output zeroed in-kernel (caller sync words), TAPS and
# ROW row pairs (C_o <= 64), ROW pairs with an odd output height
sync = torch.zeros(2, dtype=torch.int64, device=d)
for m, n, k in [(256, 300, 96), (128, 1024, 2048)]:
    a = torch.rand(m, k, device=d)
    w = torch.rand(k, n, device=d)
    pk = lcnn.pack_fc_weights(w.reshape(-1), k, n, lcnn.TF32)
    y = lcnn.fc_forward_packed(a.reshape(-1), t.NCHW, pk, m, n, k, lcnn.TF32, sync=sync)
    assert torch.allclose(y.view(m, n), a @ w, rtol=1e-2, atol=1e-2)
x = torch.rand(13 * 13 * 64 * 32, device=d)
f = torch.rand(96, 64, 3, 3, device=d)
xt = lcnn.DeviceTensor4D(32, 64, 13, 13, t.CHWN, x)
pk = lcnn.pack_conv_filters(xt, f, 96, 3, 3, 1, 1, lcnn.TF32)
lcnn.conv_forward_packed(xt, pk, 96, 3, 3, 1, 1, lcnn.TF32, sync=sync)
torch.cuda.synchronize()
assert int(sync.abs().sum()) == 0
for c in [(128, 3, 33, 33, 64, 3, 1, 1), (128, 32, 91, 91, 48, 3, 1, 1)]:
    t._check_conv(d, *c, t.CHWN, lcnn.TF32)
# round 2, later: ROW row pairs with quad-chunk TMA stores (whole tiles and a
# stream-K tail), TAPS row pairs with the 2x2 max pool in the epilogue
for c in [(64, 3, 40, 40, 64, 3, 1, 1), (128, 3, 24, 24, 64, 3, 1, 1)]:
    t._check_conv(d, *c, t.CHWN, lcnn.TF32)
tp._run(d, (32, 32, 182, 182, 64, 3, 1, 1, 2, 2))
# TAPS with two accumulators (C_o > 64 row pairs), plain and with the fused pool
t._check_conv(d, 32, 32, 182, 182, 128, 3, 1, 1, t.CHWN, lcnn.TF32)
tp._run(d, (32, 32, 182, 182, 128, 3, 1, 1, 2, 2))
print("ok")
