"""Batch sharding across GPUs (P:164 multi-GPU inference).

The encoder forward is row-independent (per-row activation quantization keeps
even the int8 path batch-invariant), so data parallelism needs no collective
inside the forward: each rank runs whole request batches on its own GPU with
replicated weights, and the only exchange is a gather of the fp32 logits
[B_local, C] to rank 0 (NCCL on GPUs, gloo in the CPU tests).

* ``shard_range``: contiguous assignment of a global batch to ranks (S:441
  "N contiguous shards"), sizes differ by at most one.
* ``ShardedEncoder``: wraps any ``encode(ids, mask) -> logits`` (the C-ABI
  encoder on a GPU, a stub on CPU) and returns the gathered logits on rank 0
  in the original order.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, stop) of rank's contiguous share of `total` items."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class ShardedEncoder:
    """Data-parallel wrapper: rank r encodes rows shard_range(B, world, r) of a
    global batch; ``encode_global`` gathers the logits to rank 0."""

    def __init__(self, encode: Callable, group=None):
        import torch.distributed as dist
        self.encode = encode
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def encode_global(self, ids, mask) -> Optional[object]:
        """ids, mask: the FULL global batch [B, S] (every rank holds it, as in a
        replicated request queue); returns logits [B, C] on rank 0, None elsewhere."""
        import torch
        import torch.distributed as dist
        B = ids.shape[0]
        lo, hi = shard_range(B, self.world, self.rank)
        local = self.encode(ids[lo:hi].contiguous(), mask[lo:hi].contiguous())
        if self.world == 1:
            return local
        C = local.shape[1]
        # gather needs equal shapes: pad every shard to the largest size
        cap = shard_range(B, self.world, 0)[1]
        buf = torch.zeros((cap, C), dtype=local.dtype, device=local.device)
        buf[: hi - lo] = local
        parts: Optional[List] = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(buf, parts, dst=0, group=self.group)
        if self.rank != 0:
            return None
        out = [parts[r][: shard_range(B, self.world, r)[1] - shard_range(B, self.world, r)[0]]
               for r in range(self.world)]
        return torch.cat(out, 0)
