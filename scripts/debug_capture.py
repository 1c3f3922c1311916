"""Why does capturing lcnn_net_forward into a CUDA graph fail?"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1610_03618_b200 import capi, netapi  # noqa: E402

text = open("configs/alexnet.json").read()
net = netapi.Network(text, 257, 32, seed=42, precision=capi.PREC_TF32)
info = net.info(1)
dev = torch.device("cuda:0")
dn, dc, dh, dw = info["dims"]
x = torch.rand(dn * dc * dh * dw, device=dev)
rows, cols = info["out"]
y = torch.empty(rows * cols, device=dev)
s = torch.cuda.current_stream()
for _ in range(3):
    net.forward(x.data_ptr(), info["first_layout"], y.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
for mode in ("global", "thread_local", "relaxed"):
    cap = torch.cuda.Stream()
    cap.wait_stream(s)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=cap, capture_error_mode=mode):
            try:
                net.forward(x.data_ptr(), info["first_layout"], y.data_ptr(), cap.cuda_stream)
            except Exception as e:
                print(mode, "forward raised:", repr(e))
                print("last_error:", capi.lib().lcnn_last_error())
                raise
        g.replay()
        torch.cuda.synchronize()
        print(mode, "capture ok")
    except Exception as e:
        print(mode, "capture failed:", repr(e)[:400])
    torch.cuda.synchronize()
