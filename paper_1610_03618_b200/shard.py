"""Batch (N) sharding across GPUs -- the only parallelism the layer path has
(SURVEY.md §8e).  Every image is independent through pooling, transforms,
softmax and convolution, so ranks never exchange activations: the data path
has no collective.  torch.distributed (NCCL on GPUs, gloo in the CPU tests) is
used only for timing (barrier, max over ranks) and for gathering the logits
rows for verification, a plain rank-order concat because classifier rows are
image-major (net.cpp:258-262)."""
from __future__ import annotations


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) images of `rank`; the first `global_batch % world` ranks
    take one extra image."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def gather_rows(local, world: int, global_rows: int | None = None):
    """All-gather every rank's row block (flat tensors) in rank order.

    With `global_rows` the blocks may be ragged as shard_range makes them
    (the first global_rows % world ranks hold one extra row): each block is
    padded to ceil(global_rows / world) rows, gathered, and trimmed back, so
    NCCL and gloo always see equal-sized buffers.  Without it every rank
    must hold the same number of elements."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    if global_rows is None:
        blocks = [(0, local.numel())] * world
        cap = local.numel()
        buf = local
    else:
        row = None
        for r in range(world):
            a, b = shard_range(global_rows, world, r)
            if r == dist.get_rank():
                if b - a and local.numel() % (b - a):
                    raise ValueError("gather_rows: local block is not whole rows")
                row = local.numel() // (b - a) if b - a else None
        # every rank needs the row width, including one holding no rows
        w = torch.tensor([row or 0], dtype=torch.int64, device=local.device)
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        row = int(w[0])
        per = -(-global_rows // world)
        cap = per * row
        blocks = [(0, (b - a) * row) for a, b in (shard_range(global_rows, world, r)
                                                  for r in range(world))]
        buf = torch.zeros(cap, dtype=local.dtype, device=local.device)
        buf[:local.numel()] = local
    out = torch.empty(world * cap, dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, buf)
    else:
        parts = list(out.view(world, -1).unbind(0))
        dist.all_gather(parts, buf)
    if global_rows is None:
        return out
    return torch.cat([out[r * cap + a:r * cap + b] for r, (a, b) in enumerate(blocks)])
