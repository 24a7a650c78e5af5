#!/usr/bin/env python3
"""Host time per public-API call inside bench.py's fresh-layout e2e stream
(configs[1]): which call blocks, and for how long."""
import collections
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

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
host_t = collections.defaultdict(float)


def call(name, fn):
    t = time.perf_counter()
    r = fn()
    host_t[name] += time.perf_counter() - t
    return r


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
    for k in (1, 2):
        ctx.stage_corpus(batches[k][0], batches[k][1], cp.vocab)
    steps, warm = 20, 3
    for s in range(warm + steps):
        if s == warm:
            if not os.environ.get("E2E_NOFETCH"):
                ctx.wait_fetch()
            host_t.clear()
            if os.environ.get("E2E_PROF"):
                ctx.set_profiling(True)
            t0 = time.perf_counter()
        call("swap_corpus", ctx.swap_corpus)
        cur, nxt = batches[(s + 1) % 4], batches[(s + 3) % 4]
        call("count", lambda: ctx.count(R.WEIGHT_TFIDF))
        call("set_reference_docs", lambda: ctx.set_reference_docs(cur[2]))
        call("sign", lambda: ctx.sign(fetch=False))
        call("stage_corpus", lambda: ctx.stage_corpus(nxt[0], nxt[1], cp.vocab))
        call("mrc_pairs_rows", lambda: ctx.mrc_pairs_rows(tau, 0, N, fetch=False))
        rowptr, cols = host[s & 1]
        if not os.environ.get("E2E_NOFETCH"):
            call("pairs_csr16_async", lambda: ctx.pairs_csr16_async(rowptr, cols))
    if not os.environ.get("E2E_NOFETCH"):
        call("wait_fetch", ctx.wait_fetch)
    t1 = time.perf_counter()
    ctx.swap_corpus()
    ctx.swap_corpus()
ph = ctx.phase_times() if os.environ.get("E2E_PROF") else {}
print(json.dumps({"phase_ms_per_batch": {k: round(v[0] / steps, 4) for k, v in ph.items() if v[1]},
                  "ms_per_batch": (t1 - t0) * 1e3 / steps,
                  "host_ms_per_call": {k: round(v * 1e3 / steps, 4) for k, v in host_t.items()}}))
