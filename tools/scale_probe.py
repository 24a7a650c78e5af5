#!/usr/bin/env python3
"""K1/K2/K3 at a larger config (default configs[3]: 200k docs, V=500k, K=64):
per-phase device times, K2 with a cold L2 (the HBM roofline), and K3 on a
row panel of the triangle.

  python tools/scale_probe.py [--config c3] [--rows 8192] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    cp, cfg = C.config_corpus(args.config)
    thr = C.load_configs()["thresholds"]
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    N, K = cp.n_docs, cfg["K"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    ctx = R.Context(0)
    ctx.set_stream(stream.cuda_stream)
    tok = torch.from_numpy(cp.tokens.view(np.int32)).to(dev)
    ctx.load_corpus_device(tok.data_ptr(), cp.doc_off, cp.vocab)
    flush = torch.empty(512 << 18, dtype=torch.int32, device=dev)
    res = {"config": args.config, "n_docs": N, "tokens": int(cp.doc_off[-1]), "K": K}
    with torch.cuda.stream(stream):
        ctx.count(R.WEIGHT_TFIDF)
        ctx.set_reference_docs(refs)
        ctx.sign(fetch=False)
        torch.cuda.synchronize()
        nnz = int(ctx.counts()[0][-1])
        ctx.set_profiling(True)
        for r in range(args.reps):
            flush.fill_(r)
            ctx.count(R.WEIGHT_TFIDF)
            ctx.set_reference_docs(refs)
            flush.fill_(r + 1)  # K2 with a cold L2
            ctx.sign(fetch=False)
        torch.cuda.synchronize()
        ph = ctx.phase_times()
        ctx.set_profiling(False)
        for k in ("count", "reference", "sign"):
            res[k + "_us"] = ph[k][0] / ph[k][1] * 1e3
        hi = min(args.rows, N)
        ctx.set_profiling(True)
        for r in range(2):
            flush.fill_(r)
            n = ctx.mrc_pairs_rows(thr["tau_mrc"], 0, hi, fetch=False)
        torch.cuda.synchronize()
        ph = ctx.phase_times()
        ctx.set_profiling(False)
        pairs = sum(N - 1 - i for i in range(hi))
        t3 = ph["pair_tiles"][0] / ph["pair_tiles"][1] * 1e-3
        res.update({"k3_rows": hi, "k3_pairs": pairs, "k3_us": t3 * 1e6, "k3_candidates": int(n),
                    "k3_tflops": 2 * K * pairs / t3 / 1e12,
                    "emit_us": ph["pair_emit"][0] / ph["pair_emit"][1] * 1e3})
    res["nnz"] = nnz
    if nnz:
        res["sign_GBps"] = (8 * nnz + (4 * K + 4) * N) / (res["sign_us"] * 1e-6) / 1e9
        res["count_GBps"] = (4 * res["tokens"] + 8 * nnz + 4 * N) / (res["count_us"] * 1e-6) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
