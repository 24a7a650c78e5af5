"""configs[4]-shaped query join (6,000-doc database, K = 128): candidate count
and hash, for comparing K3 kernel variants.  python tools/tc2_probe.py [n_queries]"""
import hashlib, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 700
cfg = C.load_configs()["configs"]["c4"]
db_spec = dict(cfg["corpus"], n_docs=6000, vocab=50000)
q_spec = dict(cfg["queries"], n_docs=nq, vocab=50000)
db = C.generate(db_spec)
q = C.generate_queries(q_spec, db_spec, db)
refs = C.sample_refs(0, db.n_docs, 128)
with R.Context(0) as dbc, R.Context(0) as qc:
    dbc.load_corpus(db.tokens, db.doc_off, db.vocab); dbc.count(); dbc.set_reference_docs(refs); dbc.sign(fetch=False)
    qc.attach_database(dbc)
    qc.load_corpus(q.tokens, q.doc_off, q.vocab); qc.count(); qc.sign(fetch=False)
    keys = qc.mrc_query_pairs(0.9)
print(len(keys), hashlib.sha256(np.ascontiguousarray(keys).tobytes()).hexdigest())
