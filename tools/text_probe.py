#!/usr/bin/env python3
"""Text front end at configs[1] scale on seeded synthetic text (one word per
token, corpus.synth_text): the command to put under ncu."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1810_03099_b200 as R  # noqa: E402
from paper_1810_03099_b200 import corpus as C  # noqa: E402

cp, cfg = C.config_corpus(sys.argv[1] if len(sys.argv) > 1 else "c1")
text, off = C.synth_text(cp.tokens, cp.doc_off, cp.vocab, 0)
ctx = R.Context(0)
ctx.load_text(text, off)
fp = ctx.simhash_text()
ctx.count(R.WEIGHT_TF)
print(len(text), "bytes", int(ctx.counts()[0][-1]), "nonzeros")
