"""The memory-bound kernels (transforms, CHWN / NCHW pooling incl. the
pipelined NCHW ring, fused and five-pass softmax) and the packed fc under
compute-sanitizer, once each at small shapes with ragged edges."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1610_03618_b200 import lcnn  # noqa: E402

rng = np.random.default_rng(0)
for (n, c, h, w) in [(32, 5, 17, 13), (64, 8, 55, 55)]:
    x = lcnn.DeviceTensor4D.from_host(rng.random(n * c * h * w, dtype=np.float32), n, c, h, w,
                                      lcnn.CHWN)
    y = lcnn.transform(x, lcnn.NCHW)
    for mode in (0, 1):
        p = lcnn.PoolParams(3, 3, 2, mode)
        lcnn.pool_layout(x, p)
        lcnn.pool_coarsened(x, p, lcnn.CoarseningPlan(2, 2))
        lcnn.pool_layout(y, p)
        lcnn.pool_coarsened_nchw(y, p, lcnn.CoarseningPlan(3, 2))
for (r, cc) in [(7, 1000), (33, 5000), (3, 20000)]:
    m = lcnn.DeviceMatrix.from_host(rng.random(r * cc, dtype=np.float32), r, cc)
    lcnn.softmax_fused(m)
    lcnn.softmax_reference(m)
wt = torch.rand(1024 * 300, device="cuda")
xt = torch.rand(64 * 1024, device="cuda")
packed = lcnn.pack_fc_weights(wt, 1024, 300)
lcnn.fc_forward_packed(xt, lcnn.NCHW, packed, 64, 300, 1024)
torch.cuda.synchronize()
print("ok")
