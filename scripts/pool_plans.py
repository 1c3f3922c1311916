"""Coarsening-plan sweep of the pooling kernels on B200 (CUDA-graph timed),
the measurement behind the autotuner's default plans."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1610_03618_b200 import capi, lcnn  # noqa: E402

dev = torch.device("cuda:0")
lib = capi.lib()


def gbs(layout, n, c, hw, win, s, fh, fw, K=50):
    x = torch.rand(n * c * hw * hw, device=dev)
    ho = (hw - win) // s + 1
    y = torch.empty(n * c * ho * ho, device=dev)
    fn = lib.lcnn_pool_coarsened if layout == capi.CHWN else None

    def launch(st):
        if layout == capi.CHWN:
            capi.check(lib.lcnn_pool_coarsened(x.data_ptr(), y.data_ptr(), n, c, hw, hw, layout, win,
                                               win, s, 0, fh, fw, None, st))
        else:
            capi.check(lib.lcnn_pool_coarsened_nchw(x.data_ptr(), y.data_ptr(), n, c, hw, hw, win,
                                                    win, s, 0, fh, fw, None, st))
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cap):
        for _ in range(K):
            launch(torch.cuda.current_stream().cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    return round((x.numel() + y.numel()) * 4 / ms / 1e6, 1)


out = {}
only = sys.argv[1:]
shapes = {"PL5": (128, 96, 55, 3, 2), "VGG1": (256, 64, 224, 2, 2), "PL7": (128, 256, 13, 3, 2)}
if "vgg" in only:
    shapes = {"VGG1": (256, 64, 224, 2, 2), "VGG2": (256, 128, 112, 2, 2),
              "VGG3": (256, 256, 56, 2, 2), "VGG4": (256, 512, 28, 2, 2),
              "VGG5": (256, 512, 14, 2, 2)}
for name, (n, c, hw, win, s) in shapes.items():
    for fh, fw in [(1, 1), (1, 2), (2, 1), (2, 2), (1, 3), (3, 1), (1, 4), (4, 1), (2, 4), (4, 2)]:
        if "nchw" not in only:
            out[f"{name}_chwn_{fh}x{fw}"] = gbs(capi.CHWN, n, c, hw, win, s, fh, fw)
    for fh, fw in [(1, 1), (2, 1), (3, 1), (4, 1), (1, 2), (2, 2), (3, 2), (4, 2)]:
        if name.startswith("VGG") and (fh, fw) == (3, 2):
            continue  # no 2x2/s2 FH=3 FW=2 instantiation
        out[f"{name}_nchw_{fh}x{fw}"] = gbs(capi.NCHW, n, c, hw, win, s, fh, fw)
print(json.dumps(out, indent=1))
