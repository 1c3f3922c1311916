import torch, json
d = torch.device("cuda:0")
n = 1640 * 2**20 // 4
x = torch.empty(n, device=d)
y = torch.empty(n, device=d)
res = {}
def t(f, bytes_, reps=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return round(bytes_ / (ms / 1e3) / 1e9, 1)
res["memset_zero_GBps"] = t(lambda: x.zero_(), n * 4)
res["fill_GBps"] = t(lambda: x.fill_(1.5), n * 4)
res["copy_rw_GBps"] = t(lambda: y.copy_(x), 2 * n * 4)
res["sum_read_GBps"] = t(lambda: x.sum(), n * 4)
print(json.dumps(res))
