#!/usr/bin/env python3
"""Run the bench step (configs[1] MRC pipeline, plus optional Simhash/Hamming
and exact pairs) a few times with no CPU baseline or e2e leg: the short,
deterministic command to put under ncu.

  python tools/prof_pipeline.py [--steps 2] [--config c1] [--simhash] [--exact]
"""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--simhash", action="store_true")
    ap.add_argument("--exact", action="store_true")
    args = ap.parse_args()
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    cp, cfg = C.config_corpus(args.config)
    thr = C.load_configs()["thresholds"]
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = R.Context(0)
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    for _ in range(args.steps):
        ctx.count(R.WEIGHT_TFIDF)
        ctx.set_reference_docs(refs)
        ctx.sign(fetch=False)
        n = ctx.mrc_pairs(thr["tau_mrc"], fetch=False)
        if args.simhash:
            ctx.simhash(0, fetch=False)
            h = ctx.hamming_pairs(thr["hamming_max"], fetch=False)
        if args.exact:
            e = ctx.exact_pairs(thr["tau_cos"], fetch=False)
    ctx.synchronize()
    print("pairs", n, "hamming", h if args.simhash else "-", "exact", e if args.exact else "-")


if __name__ == "__main__":
    main()
