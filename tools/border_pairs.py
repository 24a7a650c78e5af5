#!/usr/bin/env python3
"""List the border pairs (north_star: candidate sets identical "except for pairs
within 1e-5 of the threshold, which are listed") of the GPU compare against
the oracle: every pair the two decide differently, with the oracle's fp64
score, plus the size of the oracle's 1e-5 band.

  python tools/border_pairs.py --config c1 --out profiles/border_c1_r02.json
  python tools/border_pairs.py --config c3 --rows 2048 --out profiles/border_c3_r02.json

Test infrastructure: runs the oracle (oracle/) as the checker."""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--rows", type=int, default=0, help="row panel [0, rows) x all j > i (0: whole triangle)")
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import oracle
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C
    from tests.parity_util import BAND, assert_pairs_match, border_listing

    cp, cfg = C.config_corpus(args.config)
    K = cfg["K"]
    tau = C.load_configs()["thresholds"]["tau_mrc"] if args.tau is None else args.tau
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, K)
    N = cp.n_docs
    rows = args.rows or N
    out = {"config": args.config, "n_docs": N, "K": K, "tau": tau, "band": BAND, "rows": [0, rows], "paths": {}}
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
    pairs, border = oracle.mrc_pairs(o.S, tau, BAND, 0, rows)
    out["oracle_pairs"] = int(len(pairs))
    out["oracle_band_pairs"] = int(len(border))
    for name, path in (("tensor", R.K3_TENSOR), ("fp32", R.K3_FP32)):
        with R.Context(0) as ctx:
            ctx.set_k3_path(path)
            ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
            ctx.count()
            ctx.set_reference_docs(refs)
            ctx.sign(fetch=False)
            t = time.time()
            keys = ctx.mrc_pairs_rows(tau, 0, rows) if rows < N else ctx.mrc_pairs(tau)
            nb = assert_pairs_match(keys, pairs, border, f"{args.config} {name}")
            lst = border_listing(keys, pairs, border, o.S, tau=tau)
            assert all(abs(r["score_minus_tau"]) <= BAND for r in lst)
            out["paths"][name] = {"gpu_pairs": int(len(keys)), "disagreements": nb,
                                  "max_abs_score_minus_tau": max([abs(r["score_minus_tau"]) for r in lst], default=0.0),
                                  "pairs": lst}
            print(f"{args.config} {name}: {len(keys)} GPU pairs, {len(pairs)} oracle, {len(border)} in band, "
                  f"{nb} differ ({time.time() - t:.1f}s)", file=sys.stderr)
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
