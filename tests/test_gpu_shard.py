"""World-size-2 N-sharding of the CUDA layer path, two ranks on
cuda:0 over gloo (the gpurun box has one GPU; NCCL refuses two ranks on one
device).  Each rank runs ITS images through liblcnn_cuda.so -- VGG-style
2x2/s2 pooling in CHWN with the benched plan (1,1) and in NCHW with a
coarsened plan, AlexNet 3x3/s2 pooling, and the fused classifier -- and the
rank-order gather (ragged shards included) must be bit-equal to the
unsharded CUDA run and to the reference-pinned oracle.  This is the property
the strong-scaling bench rests on (test_conv.cpp:117-141: batch
independence)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        from oracle.oracle import CHWN, NCHW, C, approx_equal, bit_equal, rng_uniform
        from paper_1610_03618_b200 import capi, lcnn
        from paper_1610_03618_b200.shard import gather_rows, shard_range

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        assert capi.lib().lcnn_device_ok() == 1
        dev = torch.device("cuda:0")
        for (n, c, h, win, s, plan) in ((7, 64, 32, 2, 2, (1, 1)), (9, 96, 55, 3, 2, (2, 2)),
                                        (256, 16, 14, 2, 2, (1, 1))):
            p = lcnn.PoolParams(win, win, s, lcnn.MAX)
            ho = (h - win) // s + 1
            x = rng_uniform(100 + n, n * c * h * h)  # NCHW, image-contiguous
            a, b = shard_range(n, world, rank)
            xs = x.reshape(n, -1)[a:b].reshape(-1)
            # NCHW shard through the coarsened NCHW kernel
            t = lcnn.DeviceTensor4D.from_host(xs, b - a, c, h, h, NCHW, device=dev)
            y, _ = lcnn.pool_coarsened_nchw(t, p, lcnn.CoarseningPlan(2, 1))
            got = gather_rows(torch.from_numpy(y.to_host()), world, n).numpy()
            want, _ = C.pool_plain(x, n, c, h, h, NCHW, win, win, s, False)
            assert bit_equal(got, want), ("nchw", n, c, h)
            # CHWN shard: the shard's own CHWN tensor (batch axis sliced)
            xc = C.transform(xs, b - a, c, h, h, NCHW, CHWN)
            t = lcnn.DeviceTensor4D.from_host(xc, b - a, c, h, h, CHWN, device=dev)
            y, _ = lcnn.pool_coarsened(t, p, lcnn.CoarseningPlan(*plan))
            yn = lcnn.transform(y, NCHW).to_host()
            got = gather_rows(torch.from_numpy(yn), world, n).numpy()
            assert bit_equal(got, want), ("chwn", n, c, h)
            # the unsharded CUDA run agrees too
            if rank == 0:
                t = lcnn.DeviceTensor4D.from_host(x, n, c, h, h, NCHW, device=dev)
                full, _ = lcnn.pool_layout(t, p)
                assert bit_equal(full.to_host(), want)
                assert ho > 0
        # classifier rows (ragged: 5 rows over 2 ranks)
        rows, cols = 5, 1000
        z = rng_uniform(77, rows * cols, -5, 5)
        a, b = shard_range(rows, world, rank)
        m = lcnn.DeviceMatrix.from_host(z.reshape(rows, cols)[a:b].reshape(-1), b - a, cols,
                                        device=dev)
        out, _ = lcnn.softmax_fused(m)
        got = gather_rows(torch.from_numpy(out.to_host().reshape(-1)), world, rows).numpy()
        assert approx_equal(got, C.softmax_fused(z, rows, cols)[0], 1e-6)
        torch.cuda.synchronize()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()[-1500:]))


def test_two_rank_cuda_sharding_matches_unsharded(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
