"""Batch sharding across GPUs (P:164 multi-GPU inference).

The encoder forward is row-independent (per-row activation quantization keeps
even the int8 path batch-invariant), so data parallelism needs no collective
inside the forward: each rank runs its share of the request batch on its own
GPU with replicated weights, and the only exchange is a gather of the fp32
logits [B_local, C] to rank 0 (NCCL on GPUs, gloo in the CPU tests).

* ``shard_range``: contiguous assignment of a global batch to ranks (S:441
  "N contiguous shards"), sizes differ by at most one; a rank may get an empty
  shard when B < world.
* ``ShardedEncoder``: wraps an ``encode(ids, mask, out)`` that writes logits
  into ``out`` (the C-ABI ``Encoder.encode`` on a GPU, a stub on CPU).
  ``submit`` encodes this rank's shard on the caller's stream and starts the
  gather to rank 0 on a side stream, so the gather of batch k overlaps the
  forward of batch k+1; buffers are preallocated and double-buffered (no
  allocation, no ``cat`` per step).  ``Pending.result()`` returns the logits
  [B, C] in the original order on rank 0 (``None`` elsewhere).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, stop) of rank's contiguous share of `total` items."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class Pending:
    """One in-flight sharded batch: its gather handle and output slot."""

    def __init__(self, owner: "ShardedEncoder", slot: int, B: int, work):
        self.owner, self.slot, self.B, self.work = owner, slot, B, work
        self._done = False

    def wait(self):
        """Order the caller's stream after the gather (host wait on gloo)."""
        if not self._done:
            if self.work is not None:
                self.work.wait()
            self._done = True

    def result(self):
        """Logits [B, C] of the global batch on rank 0 (a view of a preallocated
        buffer, valid until this slot is reused), None on other ranks."""
        self.wait()
        o = self.owner
        if o.rank != 0:
            return None
        if not o.collective:
            return o.local[self.slot][: self.B]
        out = o.out[self.slot][: self.B]
        o._torch.index_select(o.gathered[self.slot], 0, o._index(self.B), out=out)
        return out


class ShardedEncoder:
    """Data-parallel wrapper: rank r encodes rows shard_range(B, world, r) of a
    global batch and the logits are gathered to rank 0.

    encode(ids, mask, out): writes the logits of ids / mask [b, S] into out [b, C]
    num_classes, max_batch: C and the largest global batch B (buffer sizes)
    device: where the buffers live (a CUDA device -> the gather runs on a side
    stream; CPU -> gloo, synchronous gather)."""

    def __init__(self, encode: Callable, num_classes: int, max_batch: int, device=None, group=None, depth: int = 2):
        import torch
        import torch.distributed as dist
        self._torch = torch
        self.encode, self.group, self.C = encode, group, num_classes
        # with a process group the gather runs even at world size 1 (the path the
        # GPU test exercises on one device); without one this is a plain wrapper
        self.collective = dist.is_initialized()
        self.world = dist.get_world_size(group) if self.collective else 1
        self.rank = dist.get_rank(group) if self.collective else 0
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.cuda = self.device.type == "cuda"
        self.cap = max(1, -(-max_batch // self.world))  # rows per rank slot (largest shard)
        self.max_batch = max_batch
        self.depth = depth
        kw = dict(dtype=torch.float32, device=self.device)
        self.local = [torch.zeros((self.cap, num_classes), **kw) for _ in range(depth)]
        root = self.rank == 0 and self.collective
        self.gathered = [torch.zeros((self.world * self.cap, num_classes), **kw) for _ in range(depth)] if root else None
        self.out = [torch.empty((max_batch, num_classes), **kw) for _ in range(depth)] if root else None
        self.side = torch.cuda.Stream(self.device) if self.cuda and self.collective else None
        self.inflight = [None] * depth
        self.slot = 0
        self._idx = {}

    def _index(self, B: int):
        """Rows of the gathered [world * cap, C] buffer holding the global batch, in order."""
        idx = self._idx.get(B)
        if idx is None:
            rows = []
            for r in range(self.world):
                lo, hi = shard_range(B, self.world, r)
                rows.extend(range(r * self.cap, r * self.cap + hi - lo))
            idx = self._torch.tensor(rows, dtype=self._torch.long, device=self.device)
            self._idx[B] = idx
        return idx

    def submit(self, ids, mask) -> Pending:
        """ids, mask: the FULL global batch [B, S] (every rank holds it, as in a
        replicated request queue).  Encodes this rank's shard on the current
        stream and starts the gather; returns without waiting."""
        import torch.distributed as dist
        B = ids.shape[0]
        if B > self.max_batch:
            raise ValueError(f"global batch {B} > max_batch {self.max_batch}")
        slot = self.slot
        self.slot = (slot + 1) % self.depth
        prev = self.inflight[slot]
        if prev is not None:  # the gather that last read this slot must finish before it is overwritten
            prev.wait()
        lo, hi = shard_range(B, self.world, self.rank)
        if hi > lo:  # an empty shard (B < world) still joins the gather with padding rows
            self.encode(ids[lo:hi], mask[lo:hi], self.local[slot][: hi - lo])
        work = None
        if self.collective:
            parts = list(self.gathered[slot].chunk(self.world)) if self.rank == 0 else None
            if self.cuda:
                torch = self._torch
                cur = torch.cuda.current_stream(self.device)
                self.side.wait_stream(cur)
                with torch.cuda.stream(self.side):
                    work = dist.gather(self.local[slot], parts, dst=0, group=self.group, async_op=True)
            else:
                work = dist.gather(self.local[slot], parts, dst=0, group=self.group, async_op=True)
        p = Pending(self, slot, B, work)
        self.inflight[slot] = p
        return p

    def encode_global(self, ids, mask) -> Optional[object]:
        """Synchronous convenience form: submit + result (a copy on rank 0)."""
        r = self.submit(ids, mask).result()
        return None if r is None else r.clone()
