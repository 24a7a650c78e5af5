"""H2D of one configs[1] token batch (27.2 MB pinned) as 1, 2 or 4 concurrent copies on separate
streams: does splitting the upload over copy engines beat one copy? (measured: no, 52.9 / 52.3 / 51.1 GB/s)."""
import torch, time, json
dev = torch.device("cuda", 0)
n = 27194520 // 4
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device=dev)
out = {}
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream(dev) for _ in range(parts)]
    chunk = (n + parts - 1) // parts
    best = 1e9
    for rep in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            lo, hi = i * chunk, min(n, (i + 1) * chunk)
            with torch.cuda.stream(s):
                d[lo:hi].copy_(h[lo:hi], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    out[parts] = {"ms": best * 1e3, "GBps": 4 * n / best / 1e9}
print(json.dumps(out))
