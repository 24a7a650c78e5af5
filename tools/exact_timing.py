#!/usr/bin/env python3
"""K5 exact_pairs (tau_cos) and evaluate() at configs[1]: host wall time per call."""
import json, os, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cp, cfg = C.config_corpus(sys.argv[1] if len(sys.argv) > 1 else "c1")
tau = C.load_configs()["thresholds"]["tau_cos"]
with R.Context(0) as ctx:
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"]))
    ctx.sign(fetch=False)
    ctx.simhash(0)
    out = {}
    for name, fn in (("exact_pairs", lambda: ctx.exact_pairs(tau, fetch=False)), ("evaluate", ctx.evaluate)):
        fn()
        ctx.set_profiling(True)
        t0 = time.perf_counter()
        r = fn()
        t = time.perf_counter() - t0
        ph = ctx.phase_times()
        ctx.set_profiling(False)
        out[name] = {"ms": t * 1e3, "pair_tiles_ms": ph["pair_tiles"][0], "result": r if name == "exact_pairs" else r["mrc_mae"]}
print(json.dumps(out))
