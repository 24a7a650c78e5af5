import sys; sys.path.insert(0,'/root/repo')
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cp, cfg = C.config_corpus('c1'); thr = C.load_configs()["thresholds"]
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
ctx = R.Context(0); ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
ctx.count(R.WEIGHT_TFIDF); ctx.set_reference_docs(refs); ctx.sign(fetch=False)
for _ in range(3): ctx.mrc_pairs(thr["tau_mrc"], fetch=False)
