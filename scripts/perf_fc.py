"""fc-layer probe: packed-weight tcgen05 fc at the AlexNet shapes (batch 128),
CUDA events around K launches queued behind a sleep kernel (device time
only), per-launch average.  LCNN_TC_PROBE splits operand delivery / MMA /
epilogue time."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1610_03618_b200 import lcnn  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for name, (k, n) in {"fc6": (9216, 4096), "fc7": (4096, 4096), "fc8": (4096, 1000)}.items():
    m = 128
    x = torch.rand(k * m, device=dev)
    w = torch.rand(k * n, device=dev)
    pk = lcnn.pack_fc_weights(w, k, n, lcnn.TF32)
    y = torch.empty(m * n, device=dev)
    for layout in (lcnn.CHWN, lcnn.NCHW):
        run = lambda: lcnn.fc_forward_packed(x, layout, pk, m, n, k, lcnn.TF32, out=y)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        K = 20
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            run()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / K
        res[f"{name}_{'chwn' if layout == lcnn.CHWN else 'nchw'}"] = {
            "us": round(us, 1), "weight_GBps": round(k * n * 4 / us / 1e3, 1)}
print(json.dumps(res))
