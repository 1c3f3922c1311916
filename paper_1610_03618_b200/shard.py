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


def gather_rows(local, world: int):
    """All-gather equal-sized row blocks (flat tensors) in rank order."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local)
    else:
        parts = list(out.view(world, -1).unbind(0))
        dist.all_gather(parts, local)
    return out
