#!/usr/bin/env python3
"""Breakdown of the fresh-layout e2e stream (bench.py measure_e2e_stream):
host wall time of each call of the per-batch sequence (no extra syncs)."""
import os, sys, time
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch
import bench
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C

cp, cfg = C.config_corpus("c1")
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
N = cp.n_docs
batches = bench.permuted_batches(cp, refs, 4)
ctx = R.Context(0)
rowptr = torch.empty(N + 1, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
cols = torch.empty(12_000_000, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
ctx.load_corpus(batches[0][0], batches[0][1], cp.vocab)
ctx.stage_corpus(batches[1][0], batches[1][1], cp.vocab)
names = ["swap", "stage", "count", "ref", "sign", "pairs", "csr16"]
acc = np.zeros(len(names))
for s in range(14):
    cur, nxt = batches[(s + 1) % 4], batches[(s + 2) % 4]
    t = [time.perf_counter()]
    ctx.swap_corpus(); t.append(time.perf_counter())
    ctx.stage_corpus(nxt[0], nxt[1], cp.vocab); t.append(time.perf_counter())
    ctx.count(); t.append(time.perf_counter())
    ctx.set_reference_docs(cur[2]); t.append(time.perf_counter())
    ctx.sign(fetch=False); t.append(time.perf_counter())
    ctx.mrc_pairs_rows(0.99, 0, N, fetch=False); t.append(time.perf_counter())
    ctx.wait_fetch(); ctx.pairs_csr16_async(rowptr, cols); t.append(time.perf_counter())
    if s >= 4:
        acc += np.diff(t) * 1e3
print({n: round(v / 10, 3) for n, v in zip(names, acc)}, "total", round(acc.sum() / 10, 3), "ms/batch")
