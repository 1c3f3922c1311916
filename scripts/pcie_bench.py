"""Pinned host <-> HBM copy bandwidth on the box (what bounds every e2e number):
one 2 GiB H2D, the same split over 2 / 4 streams, H2D with a concurrent D2H,
and cudaHostRegister'ed vs cudaHostAlloc'ed memory."""
import json

import torch

dev = torch.device("cuda:0")
n = 2 << 30
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device=dev)
h2 = torch.empty(n // 8, dtype=torch.float32).pin_memory()
d2 = torch.empty(n // 8, dtype=torch.float32, device=dev)
res = {}


def timed(fn, nbytes, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    return round(best, 2)


res["h2d_1stream"] = timed(lambda: d.copy_(h, non_blocking=True), n)
res["d2h_1stream"] = timed(lambda: h.copy_(d, non_blocking=True), n)
for k in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    cur = torch.cuda.current_stream()

    def split(k=k, ss=ss, cur=cur):
        m = n // 4 // k
        for i, s in enumerate(ss):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * m:(i + 1) * m].copy_(h[i * m:(i + 1) * m], non_blocking=True)
        for s in ss:
            cur.wait_stream(s)
    res[f"h2d_{k}streams"] = timed(split, n)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()


def duplex():
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


res["h2d_with_concurrent_d2h_of_1GiB(total GB/s)"] = timed(duplex, n + n // 2)
print(json.dumps(res))
