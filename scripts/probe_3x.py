import sys, torch
sys.path.insert(0, '.')
from paper_1610_03618_b200 import lcnn
dev = torch.device('cuda:0')
for k in (128, 256, 512, 1024, 2048, 4096):
    g = torch.Generator(device=dev).manual_seed(k)
    m, n = 128, 256
    a = torch.rand(m, k, device=dev, generator=g) * 2 - 1
    b = torch.rand(k, n, device=dev, generator=g) * 2 - 1
    want = a.double() @ b.double()
    r = {}
    for p in (0, 1, 2):
        got = lcnn.gemm(a.reshape(-1), b.reshape(-1), m, n, k, p).view(m, n).double()
        r[p] = got
        print(k, p, float((got - want).abs().max()))
    print(k, 'tf32 vs 3x max diff', float((r[0] - r[1]).abs().max()))
