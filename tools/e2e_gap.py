"""Where the end-to-end (host buffers) time per C3 step goes beyond the
device-timed forward: back-to-back loops of (a) ff_encode on device buffers,
(b) ff_encode_host_async, (c) (b) without distinct output buffers; wall clock
per step vs the sum of per-step CUDA-event times.  python tools/e2e_gap.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2010_13382_b200 import synth  # noqa: E402
from paper_2010_13382_b200.fastformers import Encoder  # noqa: E402

cfg = synth.config("c3").with_dtype(1)
enc = Encoder(cfg, synth.make_weights(cfg), device=0)
ids, mask = synth.make_inputs(cfg)
dids, dmask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
hids, hmask = torch.from_numpy(ids).pin_memory(), torch.from_numpy(mask).pin_memory()
N = 50
outs = [torch.empty((ids.shape[0], cfg.num_classes), dtype=torch.float32).pin_memory() for _ in range(N)]
logits = torch.empty((ids.shape[0], cfg.num_classes), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for _ in range(5):
    enc.encode(dids, dmask, logits)
    enc.encode_host_async(hids, hmask, outs[0])
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
t0 = time.perf_counter()
for k in range(N):
    ev[k][0].record(st)
    enc.encode(dids, dmask, logits)
    ev[k][1].record(st)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
evsum = sum(a.elapsed_time(b) for a, b in ev) / N
print(f"device loop: wall {wall:.4f} ms/step, event-summed {evsum:.4f} ms/step")
for name, same in (("host async, per-step outputs", False), ("host async, one output", True)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        enc.encode_host_async(hids, hmask, outs[0 if same else k])
    torch.cuda.synchronize()
    print(f"{name}: wall {(time.perf_counter() - t0) / N * 1e3:.4f} ms/step")
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(N):
    enc.encode(dids, dmask, logits)
torch.cuda.synchronize()
print(f"device loop without events: wall {(time.perf_counter() - t0) / N * 1e3:.4f} ms/step")
