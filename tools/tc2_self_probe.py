"""MRC self-join candidates (two thresholds) of a config slice at a K: counts
and a hash, for comparing K3 kernel variants (tests/test_gpu_parity_bigk.py).

  python tools/tc2_self_probe.py <config> [n_docs] [K]"""
import hashlib, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
K = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cp, cfg = C.config_corpus(name)
if n: cp = cp.slice_docs(n)
K = K or cfg["K"]
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, K)
with R.Context(0) as c:
    c.load_corpus(cp.tokens, cp.doc_off, cp.vocab); c.count(); c.set_reference_docs(refs); c.sign(fetch=False)
    h = hashlib.sha256()
    for tau in (0.9, 0.99):
        k = c.mrc_pairs(tau); h.update(np.ascontiguousarray(k).tobytes()); print(len(k))
print(h.hexdigest())
