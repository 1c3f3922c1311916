"""The memory-bound kernels (transforms incl. the short-side and N=1 paths,
CHWN / NCHW pooling incl. the pipelined NCHW ring and the tuner's plans,
fused and five-pass softmax, the sticky classifier) and the packed fc under
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
# short-side transposes (S = 1, 3, 8, 16; aligned and odd long sides) both ways
for (n, c, h, w) in [(1, 4, 8, 8), (3, 5, 7, 9), (8, 16, 12, 12), (16, 3, 11, 13), (8, 7, 5, 3)]:
    x = lcnn.DeviceTensor4D.from_host(rng.random(n * c * h * w, dtype=np.float32), n, c, h, w,
                                      lcnn.NCHW)
    lcnn.transform(lcnn.transform(x, lcnn.CHWN), lcnn.NCHW)
# generic permutations: batched NCHW <-> NHWC transposes, short-run CHWN <-> HWCN copies
for (n, c, h, w) in [(6, 20, 5, 7), (2, 33, 6, 6), (8, 4, 3, 5)]:
    x = lcnn.DeviceTensor4D.from_host(rng.random(n * c * h * w, dtype=np.float32), n, c, h, w,
                                      lcnn.NCHW)
    lcnn.transform_naive(lcnn.transform_naive(x, lcnn.NHWC), lcnn.NCHW)
    xc = lcnn.transform(x, lcnn.CHWN)
    lcnn.transform_naive(lcnn.transform_naive(xc, lcnn.HWCN), lcnn.CHWN)
# the pooling tuner (every candidate plan of both layouts) and a tuned launch
for layout in (lcnn.CHWN, lcnn.NCHW):
    p = lcnn.PoolParams(3, 3, 2, 0)
    plan = lcnn.pool_tune(16, 6, 27, 27, layout, p)
    x = lcnn.DeviceTensor4D.from_host(rng.random(16 * 6 * 27 * 27, dtype=np.float32), 16, 6, 27,
                                      27, layout)
    lcnn.pool_run_plan(x, p, plan)
for (r, cc) in [(7, 1000), (33, 5000), (3, 20000), (5, 2000), (300, 20000), (160, 40000),
                (9, 10000), (4, 12288)]:
    m = lcnn.DeviceMatrix.from_host(rng.random(r * cc, dtype=np.float32), r, cc)
    lcnn.softmax_fused(m)
    lcnn.softmax_reference(m)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = lcnn.DeviceMatrix.empty(r, cc)
    lcnn.capi.call("lcnn_softmax_fused_sticky", m.ptr(), out.ptr(), r, cc, flag.data_ptr(),
                   torch.cuda.current_stream().cuda_stream)
wt = torch.rand(1024 * 300, device="cuda")
xt = torch.rand(64 * 1024, device="cuda")
packed = lcnn.pack_fc_weights(wt, 1024, 300)
lcnn.fc_forward_packed(xt, lcnn.NCHW, packed, 64, 300, 1024)
torch.cuda.synchronize()
print("ok")
