"""Debug: lcnn_net_forward_host_many vs the device-buffer forward."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.oracle import NCHW, rng_uniform  # noqa: E402
from paper_1610_03618_b200 import capi, netapi  # noqa: E402
from test_gpu_net import MINI  # noqa: E402

netapi.set_dense_precision(capi.PREC_FP32)
net = netapi.Network(json.dumps(MINI), 257, 32, seed=42)
info = net.info(NCHW)
rows, cols = info["out"]
n, c, h, w = info["dims"]
batches = [rng_uniform(100 + i, n * c * h * w) for i in range(5)]
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev).cuda_stream
want = []
for b in batches:
    dx = torch.from_numpy(b).to(dev)
    dy = torch.empty(rows * cols, device=dev)
    net.forward(dx.data_ptr(), NCHW, dy.data_ptr(), stream)
    torch.cuda.synchronize()
    want.append(dy.cpu().numpy())
# repeat device forward: deterministic?
dx = torch.from_numpy(batches[0]).to(dev)
dy = torch.empty(rows * cols, device=dev)
net.forward(dx.data_ptr(), NCHW, dy.data_ptr(), stream)
torch.cuda.synchronize()
print("device repeat equal:", np.array_equal(dy.cpu().numpy(), want[0]))
hx = [torch.from_numpy(b).pin_memory() for b in batches]
for i in range(5):
    out = torch.zeros(rows * cols).pin_memory()
    net.forward_host(hx[i].data_ptr(), NCHW, out.data_ptr())
    print("forward_host", i, np.abs(out.numpy() - want[i]).max())
hy = [torch.zeros(rows * cols).pin_memory() for _ in batches]
net.forward_host_many([t.data_ptr() for t in hx], NCHW, [t.data_ptr() for t in hy])
for i in range(5):
    d = np.abs(hy[i].numpy() - want[i])
    print("many", i, d.max(), [np.abs(hy[i].numpy() - want[j]).max() for j in range(5)])
