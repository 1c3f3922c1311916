"""Kernel timeline of AlexNet forwards under the real launch chain (PDL on):
CUPTI start/end of every kernel (torch.profiler), so the per-layer device
time, gaps and overlaps are seen without the per-layer CUDA events that
break programmatic dependent launch."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1610_03618_b200 import capi, netapi  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
text = open(os.path.join(ROOT, "configs", "alexnet.json")).read()
netapi.set_dense_precision(capi.PREC_TF32)
net = netapi.Network(text, 257, 32, seed=42)
info = net.info(1)
dev = torch.device("cuda:0")
x = torch.rand(128 * 3 * 227 * 227, device=dev) * 2 - 1
rows, cols = info["out"]
y = torch.empty(rows * cols, device=dev)
sh = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    net.forward(x.data_ptr(), info["first_layout"], y.data_ptr(), sh)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    torch.cuda._sleep(20_000_000)
    for _ in range(3):
        net.forward(x.data_ptr(), info["first_layout"], y.data_ptr(), sh)
    torch.cuda.synchronize()
ev = sorted([e for e in p.events() if e.device_type.name == "CUDA" and "sleep" not in e.name],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
rows_out = []
prev_end = None
for e in ev:
    s, t = e.time_range.start - t0, e.time_range.end - t0
    gap = None if prev_end is None else s - prev_end
    rows_out.append({"kernel": e.name[:70], "start_us": round(s, 2), "dur_us": round(t - s, 2),
                     "gap_us": None if gap is None else round(gap, 2)})
    prev_end = t
for r in rows_out:
    print(json.dumps(r))
n = len(rows_out) // 3
print(json.dumps({"kernels_per_forward": n,
                  "forward_us": round((rows_out[-1]["start_us"] + rows_out[-1]["dur_us"]
                                       - rows_out[-n]["start_us"]), 1)}))
