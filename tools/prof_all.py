#!/usr/bin/env python3
"""Every kernel of librefsig_gpu.so once at a config's scale — the short,
deterministic command to put under `ncu --set full` for per-kernel evidence.

  python tools/prof_all.py --config c1   # the step kernels + rivals, K5, evaluation, text, FP32 K3, formats
  python tools/prof_all.py --config c3   # K2 column-owner (K=64), chunked tcgen05 K3, persistent emission
  python tools/prof_all.py --config c4   # database sign (K=128), the rb=1 tcgen05 query join, Hamming scan

A warm-up pass runs first (buffers sized, caches of the host plan built); the
measured pass runs inside the NVTX range "measured", so
`ncu --nvtx --nvtx-include "measured/"` captures only it (CUB's sorts launch
several kernels per library call, so launch counts cannot be used to skip)."""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    args = ap.parse_args()
    import torch
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    thr = C.load_configs()["thresholds"]
    tau = thr["tau_mrc"]
    if args.config == "c4":
        cfg = C.load_configs()["configs"]["c4"]
        db = C.generate(cfg["corpus"])
        q = C.generate_queries(cfg["queries"], cfg["corpus"], db)
        refs = C.sample_refs(cfg["ref_seed"], db.n_docs, cfg["K"])
        dbc, qc = R.Context(0), R.Context(0)
        dbc.load_corpus(db.tokens, db.doc_off, db.vocab)
        dbc.count()
        dbc.set_reference_docs(refs)
        dbc.sign(fetch=False)
        dbc.simhash(0)
        qc.attach_database(dbc)
        for p in range(2):
            l0 = R.Context.launch_count()
            if p == 1:
                torch.cuda.nvtx.range_push("measured")
            qc.load_corpus(q.tokens, q.doc_off, q.vocab)
            qc.count()
            qc.sign(fetch=False)
            qc.mrc_query_pairs(tau, fetch=False)
            qc.simhash(0)
            qc.hamming_query_pairs(thr["hamming_max"], fetch=False)
            qc.synchronize()
            if p == 1:
                torch.cuda.nvtx.range_pop()
            print(f"pass {p}: {R.Context.launch_count() - l0} launches")
        return
    cp, cfg = C.config_corpus(args.config)
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = R.Context(0)
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    for p in range(2):
        l0 = R.Context.launch_count()
        if p == 1:
            torch.cuda.nvtx.range_push("measured")
        ctx.count(R.WEIGHT_TFIDF)
        ctx.set_reference_docs(refs)
        ctx.sign(fetch=False)
        ctx.mrc_pairs_rows(tau, 0, cp.n_docs, fetch=False)
        if args.config == "c1":
            ctx.set_k3_path(R.K3_FP32)
            ctx.mrc_pairs_rows(tau, 0, cp.n_docs, fetch=False)
            ctx.set_k3_path(R.K3_AUTO)
            ctx.pairs_csr16()
            ctx.mrc_pairs(tau, fetch=True)  # keys
            ctx.simhash(0)
            ctx.hamming_pairs(thr["hamming_max"], fetch=False)
            ctx.exact_pairs(thr["tau_cos"], fetch=False)
            ctx.evaluate()
            ctx.exact_pairs(thr["tau_cos"], fetch=False)
            ctx.corpus_freq()
            ctx.signature_records(1)
            ctx.pair_cosines(np.array([1, (2 << 32) | 3], np.uint64))
            ctx.counts()
        ctx.synchronize()
        if p == 1:
            torch.cuda.nvtx.range_pop()
        print(f"pass {p}: {R.Context.launch_count() - l0} launches")
    if args.config == "c1":
        text, off = C.synth_text(cp.tokens[: int(cp.doc_off[4000])], cp.doc_off[:4001], cp.vocab)
        with R.Context(0) as t:
            t.load_text(text, off)
            t.simhash_text()
    ctx.synchronize()


if __name__ == "__main__":
    main()
