#!/usr/bin/env python3
"""Pinned host<->device copy bandwidth on this box (the e2e stream's bound):
H2D of the configs[1] token array size, D2H of the CSR16 result size, and
both at once on two streams."""
import json
import time

import torch

dev = torch.device("cuda", 0)
h2d_b, d2h_b = 27194520, 14041010
hs = torch.empty(h2d_b, dtype=torch.uint8).pin_memory()
ds = torch.empty(h2d_b, dtype=torch.uint8, device=dev)
hr = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
dr = torch.empty(d2h_b, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
out = {}
for name, fn in (("h2d", lambda: ds.copy_(hs, non_blocking=True)), ("d2h", lambda: hr.copy_(dr, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    out[name] = {"ms": dt * 1e3, "GBps": (h2d_b if name == "h2d" else d2h_b) / dt / 1e9}
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    with torch.cuda.stream(s1):
        ds.copy_(hs, non_blocking=True)
    with torch.cuda.stream(s2):
        hr.copy_(dr, non_blocking=True)
torch.cuda.synchronize()
out["both_ms"] = (time.perf_counter() - t) / 20 * 1e3
print(json.dumps(out))
