#!/usr/bin/env python3
"""CUPTI timeline (torch.profiler / Kineto) of the fresh-layout e2e stream at
configs[1]: every memcpy and kernel of the library with start/end on its
stream, summarised per batch (H2D / compute / D2H intervals)."""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1810_03099_b200 as R  # noqa: E402
from paper_1810_03099_b200 import corpus as C  # noqa: E402

cp, cfg = C.config_corpus("c1")
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
tau = C.load_configs()["thresholds"]["tau_mrc"]
N = cp.n_docs
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
ctx = R.Context(0)
ctx.set_stream(stream.cuda_stream)
batches = bench.permuted_batches(cp, refs, 4)
with torch.cuda.stream(stream):
    tok, off, rf = batches[0]
    ctx.load_corpus(tok, off, cp.vocab)
    ctx.count(R.WEIGHT_TFIDF)
    ctx.set_reference_docs(rf)
    ctx.sign(fetch=False)
    cap = int(ctx.mrc_pairs_rows(tau, 0, N, fetch=False) * 1.2) + 4096
    host = [(torch.empty(N + 1, dtype=torch.int64).pin_memory().numpy().view(np.uint64),
             torch.empty(cap, dtype=torch.int16).pin_memory().numpy().view(np.uint16)) for _ in range(2)]
    torch.cuda.synchronize(dev)
    ctx.stage_corpus(batches[1][0], batches[1][1], cp.vocab)
    ctx.stage_corpus(batches[2][0], batches[2][1], cp.vocab)

    def loop(steps, s0=0):
        for s in range(s0, s0 + steps):
            ctx.swap_corpus()
            cur, nxt = batches[(s + 1) % 4], batches[(s + 3) % 4]
            ctx.count(R.WEIGHT_TFIDF)
            ctx.set_reference_docs(cur[2])
            ctx.sign(fetch=False)
            ctx.stage_corpus(nxt[0], nxt[1], cp.vocab)
            ctx.mrc_pairs_rows(tau, 0, N, fetch=False)
            rowptr, cols = host[s & 1]
            ctx.pairs_csr16_async(rowptr, cols)
    loop(4)
    ctx.wait_fetch()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        loop(6, 4)
        ctx.wait_fetch()
    torch.cuda.synchronize(dev)
path = os.path.join(REPO, "gpurun_out", "e2e_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
rows = []
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset"):
        rows.append((e["ts"], e["ts"] + e["dur"], cat, e.get("args", {}).get("stream"), e["name"][:40],
                     e.get("args", {}).get("bytes", 0)))
    elif cat == "cuda_runtime" and e["name"] in ("cudaStreamSynchronize", "cudaEventSynchronize"):
        rows.append((e["ts"], e["ts"] + e["dur"], "host_sync", None, e["name"], 0))
rows.sort()
t0 = rows[0][0]
for r in rows:
    if r[2] == "gpu_memcpy" or r[2] == "host_sync" or r[5] > 1e6 or "emit" in r[4] or "count_warp_kernel<2>" in r[4]:
        print(f"{r[0]-t0:9.1f} {r[1]-t0:9.1f} {r[1]-r[0]:7.1f} {r[2]:10s} s={r[3]} {r[4]} {r[5]}")
