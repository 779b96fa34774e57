"""a12 on the GPU: the sharded encoder (paper_2010_13382_b200/dist.py) around
the CUDA Encoder, with the logits gather running on NCCL (a world-size-1
process group on cuda:0: the same side-stream gather, double-buffered slots
and reordering the multi-GPU path uses), bit-identical to the unsharded call."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2010_13382_b200 import synth
from paper_2010_13382_b200.dist import ShardedEncoder
from paper_2010_13382_b200.fastformers import Encoder

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("name,dt", [("c1", 1), ("c3", 1), ("c3", 0)])
def test_sharded_encoder_nccl_bit_identical(nccl_group, name, dt):
    cfg = synth.config(name).with_dtype(dt)
    B_max, S = (8, 32) if name == "c1" else (48, 128)
    cfg = cfg.with_batch(B_max, S)
    w = synth.make_weights(cfg)
    enc = Encoder(cfg, w, max_tokens=B_max * S)
    sh = ShardedEncoder(lambda i, m, o: enc.encode(i, m, o), cfg.num_classes, B_max, device="cuda:0")
    batches = []
    for k, B in enumerate((B_max, 5, 1, B_max - 3)):
        ids, mask = synth.make_inputs(cfg, B=B, S=S, ragged=True, seed=400 + k)
        batches.append((torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()))
    ref = [enc.encode(i, m).clone() for i, m in batches]
    got = []
    pend = []
    for i, m in batches:  # submitted back to back: the gathers overlap the next forwards
        pend.append(sh.submit(i, m))
        if len(pend) == sh.depth:
            got.append(pend.pop(0).result().clone())
    got += [p.result().clone() for p in pend]
    torch.cuda.synchronize()
    for g, r in zip(got, ref):
        assert torch.equal(g, r)
