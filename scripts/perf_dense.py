"""Tensor-core throughput probe: tcgen05 TF32 GEMM and CHWN implicit-GEMM
conv at AlexNet shapes (CUDA events, median of 10 after warm-up)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1610_03618_b200 import lcnn  # noqa: E402

dev = torch.device("cuda:0")


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


only = sys.argv[1:]  # optional name filters, e.g. conv1_chwn


def want(name):
    return not only or any(o in name for o in only)


res = {}
for (m, n, k) in [(8192, 8192, 8192), (4096, 4096, 4096), (128, 4096, 9216), (1024, 4096, 9216)]:
    if not want(f"gemm_{m}x{n}x{k}"):
        continue
    a = torch.rand(m * k, device=dev)
    b = torch.rand(k * n, device=dev)
    c = torch.empty(m * n, device=dev)
    ws = torch.empty(1, device=dev)
    ms = timeit(lambda: lcnn.gemm(a, b, m, n, k, lcnn.TF32, out=c, workspace=ws))
    res[f"gemm_{m}x{n}x{k}"] = {"ms": round(ms, 4), "tflops": round(2 * m * n * k / ms / 1e9, 1)}
# AlexNet convs, CHWN, batch 128 (input dims = previous pool outputs)
convs = {"conv1": (3, 227, 96, 11, 4, 0), "conv2": (96, 27, 192, 5, 1, 2), "conv3": (192, 13, 384, 3, 1, 1),
         "conv4": (384, 13, 256, 3, 1, 1), "conv5": (256, 13, 256, 3, 1, 1),
         # VGG-16 shapes (run only when named: `perf_dense.py vgg`)
         "vgg1_1": (3, 224, 64, 3, 1, 1), "vgg1_2": (64, 224, 64, 3, 1, 1),
         "vgg2_1": (64, 112, 128, 3, 1, 1), "vgg2_2": (128, 112, 128, 3, 1, 1),
         "vgg3_1": (128, 56, 256, 3, 1, 1), "vgg3_2": (256, 56, 256, 3, 1, 1),
         "vgg4_2": (512, 28, 512, 3, 1, 1), "vgg5_1": (512, 14, 512, 3, 1, 1)}
N = 128
for layout, tag in ((lcnn.CHWN, "chwn"), (lcnn.NCHW, "nchw")):
    for name, (ci, hw, co, f, s, p) in convs.items():
        if not want(f"{name}_{tag}") or (name.startswith("vgg") and not only):
            continue
        x = lcnn.DeviceTensor4D(N, ci, hw, hw, layout, torch.rand(N * ci * hw * hw, device=dev))
        w = torch.rand(co * ci * f * f, device=dev)
        ho = (hw + 2 * p - f) // s + 1
        out = lcnn.DeviceTensor4D(N, co, ho, ho, layout, torch.empty(N * co * ho * ho, device=dev))
        ws = torch.empty(64 << 20, device=dev)
        ms = timeit(lambda: lcnn.conv_forward(x, w, co, f, f, s, p, lcnn.TF32, out=out, workspace=ws))
        fl = 2 * N * co * ho * ho * ci * f * f
        res[f"{name}_{tag}"] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}
print(json.dumps(res))
