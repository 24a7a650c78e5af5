#!/usr/bin/env python3
"""refsig_gpu_evaluate at configs[1] (all 177.6M pairs): host wall time per
call and the per-phase device times (exact_tail dump + evaluation tiles)."""
import json, os, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C

cp, cfg = C.config_corpus(sys.argv[1] if len(sys.argv) > 1 else "c1")
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
with R.Context(0) as ctx:
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(refs)
    ctx.sign(fetch=False)
    ctx.simhash(0)
    e = ctx.evaluate()
    ctx.set_profiling(True)
    t0 = time.perf_counter()
    e = ctx.evaluate()
    t = time.perf_counter() - t0
    ph = ctx.phase_times()
print(json.dumps({"ms": t * 1e3, "pair_tiles_ms": ph["pair_tiles"][0], **e}))
