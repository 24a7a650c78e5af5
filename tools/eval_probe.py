import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cp, cfg = C.config_corpus('c1')
refs = C.sample_refs(cfg['ref_seed'], cp.n_docs, cfg['K'])
ctx = R.Context(0)
ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
for wm in (R.WEIGHT_TF, R.WEIGHT_TFIDF):
    ctx.count(wm); ctx.set_reference_docs(refs); ctx.sign(fetch=False); ctx.simhash(0, wm)
    ctx.evaluate()
    t = time.perf_counter(); e = ctx.evaluate(); t = time.perf_counter() - t
    print(wm, round(t * 1e3, 2), 'ms', e)
