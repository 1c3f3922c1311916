"""fc-layer probe with DRAM-cold weights: the packed-weight tcgen05 fc at the
AlexNet shapes (batch 128, CHWN activations for fc6 as in the chain), the
weights rotated over enough packed copies (> 2.5x L2) that every launch
streams them from HBM, as inside the forward.  CUDA events around K launches
queued behind a sleep kernel, per-launch average.  Run under LCNN_TC_PROBE
(PROFILING build) to split loads / MMA / epilogue."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1610_03618_b200 import lcnn  # noqa: E402

dev = torch.device("cuda:0")
res = {"probe": os.environ.get("LCNN_TC_PROBE", "0"), "splitk": os.environ.get("LCNN_FC_SPLITK", "1"),
       "sync": os.environ.get("LCNN_FC_SYNC", "0")}
# LCNN_FC_SYNC=1: per-call-site sync words (lcnn_fc_forward_packed_ex), the
# stream-K output zeroed in-kernel instead of by a zeroing launch
sync = torch.zeros(2, dtype=torch.int64, device=dev) if res["sync"] == "1" else None
for name, (k, n, lay) in {"fc6": (9216, 4096, lcnn.CHWN), "fc7": (4096, 4096, lcnn.NCHW),
                          "fc8": (4096, 1000, lcnn.NCHW)}.items():
    m = 128
    x = torch.rand(k * m, device=dev)
    w = torch.rand(k * n, device=dev)
    pk0 = lcnn.pack_fc_weights(w, k, n, lcnn.TF32)
    del w
    copies = max(1, -(-320 * 2**20 // pk0.numel()))
    pks = [pk0] + [pk0.clone() for _ in range(copies - 1)]
    y = torch.empty(m * n, device=dev)
    runs = [lambda p=p: lcnn.fc_forward_packed(x, lay, p, m, n, k, lcnn.TF32, out=y, sync=sync)
            for p in pks]
    for r in runs:
        r()
    torch.cuda.synchronize()
    K = 8 * copies
    torch.cuda._sleep(20_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(K):
        runs[i % copies]()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / K
    res[name] = {"us": round(us, 2), "weight_GBps": round(k * n * 4 / us / 1e3, 1), "copies": copies}
    del pks, runs
print(json.dumps(res))
