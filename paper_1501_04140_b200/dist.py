"""Multi-GPU sharding of the encoder (DESIGN.md §"Multi-GPU").

The quadtree of each top-level B_max x B_max block depends only on that block and on the
level's domain pools, which every rank builds for itself from the full image; so ranks encode
disjoint sets of top-level blocks (t % world == rank, row-major t) with no exchange on the data
path.  The only collective gathers the finished codes once per encode (an NCCL all-gather over
NVLink when the process group is NCCL), after which fic_merge_shards restores the canonical
order (B descending, then (ry, rx)) -- identical to the single-GPU output.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .fic import RECORD_BYTES, Context


def gather_records(local, group=None):
    """All-gather variable-length uint8 [n_i, 40] record tensors -> (padded [W*stride, 40], counts).

    Works on any process-group backend (NCCL for CUDA tensors, gloo for CPU tensors)."""
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    stride = max(1, max(counts))
    pad = torch.zeros((stride, RECORD_BYTES), dtype=torch.uint8, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat(bufs, 0), counts, stride


def sharded_encode(ctx: Context, img, cfg, group=None):
    """Encode this rank's shard on its GPU, gather every shard, merge canonically (all ranks)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    local = ctx.encode_cfg(cfg, img, shard=rank, n_shards=world)
    allrec, counts, stride = gather_records(local, group)
    return ctx.merge_shards(allrec, counts, stride)


def native_context(device: int, group=None, **kw) -> Context:
    """A Context with the library's own NCCL communicator over the ranks of `group`: rank 0 makes
    the unique id, torch.distributed hands it to the others (plumbing only)."""
    from .fic import nccl_unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return Context(device, nccl=(obj[0], world, rank), **kw)


def native_sharded_encode(ctx: Context, img, cfg):
    """fic_encode_nccl (fic_encode_nccl_topk for a top-K cfg): shard, NCCL all-gather and merge
    inside the library."""
    return ctx.encode_nccl_cfg(cfg, img)
