import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cfgs = C.load_configs(); cfg, thr = cfgs["configs"]["c4"], cfgs["thresholds"]; tau = thr["tau_mrc"]
db_spec = dict(cfg["corpus"]); t=time.time(); db = C.generate(db_spec); print("gen", time.time()-t, flush=True)
qb = []
for b in range(5):
    q = C.generate_queries(dict(cfg["queries"], seed=cfg["queries"]["seed"] + b), db_spec, db)
    pin = torch.empty(len(q.tokens), dtype=torch.int32).pin_memory().numpy().view(np.uint32); pin[:] = q.tokens
    qb.append((pin, q.doc_off, q.vocab))
refs = C.sample_refs(cfg["ref_seed"], db.n_docs, cfg["K"])
dev = torch.device("cuda", 0); stream = torch.cuda.Stream(dev)
dbc = R.Context(0); qc = R.Context(0)
dbc.load_corpus(db.tokens, db.doc_off, db.vocab); dbc.count(); dbc.set_reference_docs(refs); dbc.sign(fetch=False); dbc.simhash(0); dbc.synchronize()
qc.set_stream(stream.cuda_stream); qc.attach_database(dbc)
def T(name, f, sync):
    t = time.perf_counter(); r = f()
    if sync: torch.cuda.synchronize(dev)
    print(f"  {name}: {1e3*(time.perf_counter()-t):.2f} ms", flush=True); return r
with torch.cuda.stream(stream):
    for sync in (False, True):
        print("sync" if sync else "nosync")
        qc.load_corpus(*qb[0]); qc.count(); qc.sign(fetch=False); qc.mrc_query_pairs(tau, fetch=False); qc.simhash(0); qc.hamming_query_pairs(thr["hamming_max"], fetch=False); torch.cuda.synchronize(dev)
        T("stage", lambda: qc.stage_corpus(*qb[1]), sync)
        for b in range(1, 4):
            print(" batch", b)
            T("swap", qc.swap_corpus, sync)
            if b + 1 <= 3: T("stage", lambda: qc.stage_corpus(*qb[b + 1]), sync)
            T("count", qc.count, sync)
            T("sign", lambda: qc.sign(fetch=False), sync)
            T("mrc", lambda: qc.mrc_query_pairs(tau, fetch=False), sync)
            T("simhash", lambda: qc.simhash(0), sync)
            T("ham", lambda: qc.hamming_query_pairs(thr["hamming_max"], fetch=False), sync)
        torch.cuda.synchronize(dev)
