import sys; sys.path.insert(0,'/root/repo')
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cp, cfg = C.config_corpus('c1')
ctx = R.Context(0); ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab); ctx.count(R.WEIGHT_TFIDF)
for _ in range(2): n = ctx.exact_pairs(0.8, fetch=False)
print(n)
