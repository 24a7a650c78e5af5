#!/usr/bin/env python3
"""Per-tile clock64 trace of the tcgen05 K3 kernel (k3_tc.cu) at configs[1].

Build the library with the trace compiled in, then run with REFSIG_TC_DEBUG:
    touch paper_1810_03099_b200/csrc/k3_tc.cu && make NVEXTRA=-DREFSIG_TC_TRACE all
    REFSIG_TC_DEBUG=8  python tools/tc_trace_run.py   # CTA 0
    REFSIG_TC_DEBUG=24 python tools/tc_trace_run.py   # last CTA
Bits 1/2/4 additionally skip the epilogue math / B refills / MMAs (timing
experiments only: the pairs are then wrong). The trace is printed to stderr
on the third mrc_pairs call.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_03099_b200 as R  # noqa: E402
from paper_1810_03099_b200 import corpus as C  # noqa: E402

cp, cfg = C.config_corpus("c1")
thr = C.load_configs()["thresholds"]
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
ctx = R.Context(0)
ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
ctx.count(R.WEIGHT_TFIDF)
ctx.set_reference_docs(refs)
ctx.sign(fetch=False)
for _ in range(3):
    ctx.mrc_pairs(thr["tau_mrc"], fetch=False)
