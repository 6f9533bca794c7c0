"""Raw pinned H2D bandwidth vs the end-to-end scorer at several chunk sizes (diagnostic)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2101_06354_b200 as P

dev = torch.device("cuda", 0)
n, h, w = 64, 1080, 1920
ref = torch.randint(0, 256, (n, h, w), dtype=torch.uint8).pin_memory()
dist = torch.randint(0, 256, (n, h, w), dtype=torch.uint8).pin_memory()
dref = torch.empty_like(ref, device=dev)
ddist = torch.empty_like(dist, device=dev)
for _ in range(3):
    dref.copy_(ref, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    dref.copy_(ref, non_blocking=True)
    ddist.copy_(dist, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"single-stream whole-batch H2D: {2 * ref.numel() / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        dref.copy_(ref, non_blocking=True)
    with torch.cuda.stream(s2):
        ddist.copy_(dist, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"two-stream H2D: {2 * ref.numel() / dt / 1e9:.1f} GB/s")
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
spec = P.MultiscaleSpec.product(5)
for chunk in (4, 8, 16, 32):
    sc = P.HostBatchScorer(cfg, spec, mode="both", chunk=chunk)
    for _ in range(2):
        sc(ref, dist)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        sc(ref, dist)
    dt = (time.perf_counter() - t0) / 5
    print(f"e2e chunk {chunk}: {n / dt:.0f} pairs/s ({2 * ref.numel() / dt / 1e9:.1f} GB/s of input)")
