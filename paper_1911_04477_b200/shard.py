"""Batch sharding across GPUs: contiguous shards, replicated weights, one
collective -- the final logits gather.

Images are independent in the reference (the per-image loop of conv_forward_binary,
network.cpp:71-78), so rank r of W processes images [start, start + count) of the global batch
and generates exactly those inputs at their global element offset (fill_random is
counter-based, tensor.cpp:65-96). The logits, [features, count] per rank in the reference's
[features, batch] layout (network.hpp:104-105), are all-gathered and concatenated along the
batch axis.
"""
from __future__ import annotations

IMG_ELEMS = 3 * 32 * 32


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """[start, start + count) of `rank`: ceil-split, trailing ranks may get fewer (or zero)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-global_batch // world)
    start = min(rank * per, global_batch)
    return start, min(per, global_batch - start)


def input_offset(global_batch: int, world: int, rank: int, elems_per_image: int = IMG_ELEMS) -> int:
    """Element offset of this rank's first input value in the global synthetic tensor."""
    return shard_range(global_batch, world, rank)[0] * elems_per_image


def gather_logits(local, global_batch: int, group=None):
    """All-gather every rank's [F, count] logits into the global [F, global_batch] matrix.

    Shards are padded to the common ceil size for the collective (all_gather needs equal
    shapes) and the padding is dropped after the concatenation. Works with NCCL (CUDA tensors)
    and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = -(-global_batch // world)
    F, n = local.shape
    buf = torch.zeros((F, per), dtype=local.dtype, device=local.device)
    buf[:, :n] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat([p[:, :shard_range(global_batch, world, r)[1]] for r, p in enumerate(parts)], dim=1)
    return out


def assemble_gathered(gathered):
    """[world, F, B] (all_gather_into_tensor of equal [F, B] shards, rank-major) -> the global
    [F, world*B] logits in the reference's [features, batch] layout, images in rank order."""
    world, F, B = gathered.shape
    return gathered.permute(1, 0, 2).reshape(F, world * B)
