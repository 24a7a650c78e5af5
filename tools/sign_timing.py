#!/usr/bin/env python3
"""K2 sign in isolation at a config's scale: device time per
launch with a cold L2 (512 MB flush before each launch), the SURVEY §8d
algorithmic bytes (8 nnz + 4K + 4 per signature) and the HBM roofline
fraction against MEASURED_PEAKS.json.

  python tools/sign_timing.py --config c3 [--reps 10]"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    cp, cfg = C.config_corpus(args.config)
    K = cfg["K"]
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, K)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    ctx = R.Context(0)
    ctx.set_stream(stream.cuda_stream)
    flush = torch.empty(512 << 18, dtype=torch.int32, device=dev)
    with torch.cuda.stream(stream):
        ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
        ctx.count()
        ctx.set_reference_docs(refs)
        ctx.sign(fetch=False)
        rowptr, _, _ = ctx.counts()
        nnz = int(rowptr[-1])
        ctx.set_profiling(True)
        for r in range(args.reps):
            flush.fill_(r + 7)
            ctx.sign(fetch=False)
        torch.cuda.synchronize(dev)
        ph = ctx.phase_times()
        ctx.set_profiling(False)
    t, calls = ph["sign"]
    ms = t / max(calls, 1)
    N = cp.n_docs
    nbytes = 8 * nnz + (4 * K + 4) * N
    peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6458.7))
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(json.dumps({"config": args.config, "K": K, "n_docs": N, "nnz": nnz, "ms": ms, "bytes": nbytes,
                      "GBps": gbs, "hbm_peak": hbm, "frac": gbs / hbm, "signatures_per_sec": N / (ms * 1e-3)}))


if __name__ == "__main__":
    main()
