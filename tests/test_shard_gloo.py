"""World-size-2 gloo tests (CPU) of the N>1 host logic: shard ranges, the
rank-order logits gather, max-over-ranks timing, and batch independence of
the sharded layer path (each rank pools / softmaxes its own images with the
reference-pinned oracle; the gathered result equals the unsharded run)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1610_03618_b200.shard import shard_range


def test_shard_ranges_partition():
    for n in (1, 7, 128, 256, 1023):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                a, b = shard_range(n, world, r)
                seen.extend(range(a, b))
            assert seen == list(range(n))


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

        from oracle.oracle import CHWN, NCHW, C, bit_equal, rng_uniform
        from paper_1610_03618_b200.shard import gather_rows, max_over_ranks, shard_range

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        # max over ranks
        assert max_over_ranks(10.0 + rank) == 10.0 + world - 1
        # batch independence: NCHW images are contiguous per image
        n, c, h, w = 6, 3, 13, 13
        x = rng_uniform(11, n * c * h * w).reshape(n, -1)
        a, b = shard_range(n, world, rank)
        mine, _ = C.pool_plain(x[a:b].reshape(-1), b - a, c, h, w, NCHW, 3, 3, 2, True)
        got = gather_rows(torch.from_numpy(mine), world).numpy()
        full, _ = C.pool_plain(x.reshape(-1), n, c, h, w, NCHW, 3, 3, 2, True)
        assert bit_equal(got, full)
        # softmax rows (classifier tail): gathered rows == unsharded rows
        logits = rng_uniform(12, n * 10, -5, 5).reshape(n, 10)
        mine, _ = C.softmax_fused(logits[a:b].reshape(-1), b - a, 10)
        got = gather_rows(torch.from_numpy(mine), world).numpy()
        assert bit_equal(got, C.softmax_fused(logits.reshape(-1), n, 10)[0])
        # CHWN shard built by slicing the batch axis pools to the same images
        xc = C.transform(x.reshape(-1), n, c, h, w, NCHW, CHWN).reshape(c * h * w, n)
        shard = np.ascontiguousarray(xc[:, a:b]).reshape(-1)
        out_c, _ = C.pool_plain(shard, b - a, c, h, w, CHWN, 3, 3, 2, False)
        out_n = C.transform(out_c, b - a, c, 6, 6, CHWN, NCHW)
        got = gather_rows(torch.from_numpy(out_n), world).numpy()
        assert bit_equal(got, C.pool_plain(x.reshape(-1), n, c, h, w, NCHW, 3, 3, 2, False)[0])
        # ragged shards (n % world != 0): rows are padded, gathered, trimmed
        for n_r in (7, 1, 3):
            a, b = shard_range(n_r, world, rank)
            rows = rng_uniform(13, n_r * 5, -5, 5).reshape(n_r, 5)
            mine, _ = C.softmax_fused(rows[a:b].reshape(-1), b - a, 5) if b > a else (
                np.zeros(0, np.float32), None)
            got = gather_rows(torch.from_numpy(mine), world, n_r).numpy()
            assert bit_equal(got, C.softmax_fused(rows.reshape(-1), n_r, 5)[0]), n_r
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
