"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel path:
contiguous sharding, logits gather to rank 0, and sharded == single-process
results (the oracle stands in for the per-GPU encoder)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_13382_b200.dist import ShardedEncoder, shard_range


def test_shard_range_contiguous_and_balanced():
    for total in (0, 1, 5, 10, 256, 257):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    assert [shard_range(10, 2, r) for r in range(2)] == [(0, 5), (5, 10)]  # S:443 example


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2010_13382_b200 import synth
    cfg = synth.config("c1")
    w = synth.make_weights(cfg)
    orc = oracle.Oracle(cfg, w)
    ids, mask = synth.make_inputs(cfg, B=B, ragged=True, seed=3)

    def encode(i, m):
        return torch.from_numpy(orc.encode(i.numpy(), m.numpy()))

    got = ShardedEncoder(encode).encode_global(torch.from_numpy(ids), torch.from_numpy(mask))
    if rank == 0:
        np.save(out_path, got.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [4, 5])
def test_sharded_equals_single_process_gloo(tmp_path, B):
    out = str(tmp_path / "logits.npy")
    mp.spawn(_worker, args=(2, _free_port(), B, out), nprocs=2, join=True)
    got = np.load(out)
    import oracle
    from paper_2010_13382_b200 import synth
    cfg = synth.config("c1")
    ids, mask = synth.make_inputs(cfg, B=B, ragged=True, seed=3)
    ref = oracle.Oracle(cfg, synth.make_weights(cfg)).encode(ids, mask)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)  # batch invariance makes sharding exact
