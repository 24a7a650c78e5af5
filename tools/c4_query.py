#!/usr/bin/env python3
"""configs[4] query-vs-database at full scale: a 1,000,000-document database
(K = 128) resident in HBM, and batches of 10,000 query documents streamed
through one query context (the next batch's token upload overlaps the current
batch's compute: stage_corpus / swap_corpus). Per batch: count (database IDF)
-> sign -> 10,000 x 1,000,000 MRC compare with candidate compaction -> Simhash
-> 64-bit Hamming scan (<= 3) over the same database.

  python tools/c4_query.py [--batches 4] [--db-docs 1000000]

Prints one JSON line: database build time and signatures/s, per-batch device
time (CUDA events on the query stream over the whole streamed run / batches),
query signatures/s, Q x D doc-pairs/s for the compare and for the Hamming
scan, candidates per batch, per-phase device times."""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--db-docs", type=int, default=0)
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--path", choices=["auto", "tensor", "fp32"], default="auto")
    ap.add_argument("--K", type=int, default=0, help="override configs[4]'s K (measurement)")
    args = ap.parse_args()
    import torch
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    cfg = C.load_configs()["configs"]["c4"]
    thr = C.load_configs()["thresholds"]
    tau = thr["tau_mrc"] if args.tau is None else args.tau
    db_spec = dict(cfg["corpus"])
    if args.db_docs:
        db_spec["n_docs"] = args.db_docs
    t = time.time()
    db = C.generate(db_spec)
    # query batches: the configs[4] query stream (10% near-duplicates of database docs), one seed per batch
    batches = []
    for b in range(args.batches + 1):
        qs = dict(cfg["queries"], seed=cfg["queries"]["seed"] + b)
        qb = C.generate_queries(qs, db_spec, db)
        pin = torch.empty(len(qb.tokens), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        pin[:] = qb.tokens
        batches.append((pin, qb.doc_off, qb.vocab))
    gen_s = time.time() - t
    K = args.K or cfg["K"]
    refs = C.sample_refs(cfg["ref_seed"], db.n_docs, K)
    dev = torch.device("cuda", 0)
    dbc = R.Context(0)
    qc = R.Context(0)
    stream = torch.cuda.Stream(dev)
    qc.set_stream(stream.cuda_stream)
    qc.set_k3_path({"auto": R.K3_AUTO, "tensor": R.K3_TENSOR, "fp32": R.K3_FP32}[args.path])
    # database (built once; timed with the library's phase events)
    dbc.set_profiling(True)
    t = time.time()
    dbc.load_corpus(db.tokens, db.doc_off, db.vocab)
    dbc.count()
    dbc.set_reference_docs(refs)
    dbc.sign(fetch=False)
    dbc.simhash(0)
    dbc.synchronize()
    db_wall = time.time() - t
    ph = dbc.phase_times()
    dbc.set_profiling(False)
    db_sig_ms = sum(ph[k][0] for k in ("count", "reference", "sign"))
    qc.attach_database(dbc)
    # warm-up: every batch once (sizes the streaming buffers for the largest batch, builds the
    # database column forms)
    for wb in batches:
        qc.load_corpus(*wb)
        qc.count()
        qc.sign(fetch=False)
        qc.mrc_query_pairs(tau, fetch=False)
        qc.simhash(0)
        qc.hamming_query_pairs(thr["hamming_max"], fetch=False)
    torch.cuda.synchronize(dev)
    # streamed batches
    qc.set_profiling(True)
    cands, hams = [], []
    with torch.cuda.stream(stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qc.stage_corpus(*batches[1])
        if args.batches >= 2:
            qc.stage_corpus(*batches[2])  # two batches staged ahead
        e0.record(stream)
        w0 = time.time()
        for b in range(1, args.batches + 1):
            qc.swap_corpus()
            qc.count()
            qc.sign(fetch=False)
            if b + 2 <= args.batches:
                qc.stage_corpus(*batches[b + 2])  # host plan + upload of a later batch overlap this one
            cands.append(qc.mrc_query_pairs(tau, fetch=False))
            qc.simhash(0)
            hams.append(qc.hamming_query_pairs(thr["hamming_max"], fetch=False))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.time() - w0
    ph = qc.phase_times()
    qc.set_profiling(False)
    ms_batch = e0.elapsed_time(e1) / args.batches
    Q = len(batches[1][1]) - 1
    D = db.n_docs
    sig_ms = sum(ph[k][0] for k in ("count", "sign")) / args.batches
    out = {"config": "c4", "db_docs": D, "queries_per_batch": Q, "K": K, "tau": tau, "batches": args.batches,
           "generate_s": gen_s, "db_build_wall_s": db_wall, "db_signature_ms": db_sig_ms,
           "db_signatures_per_sec": D / (db_sig_ms * 1e-3),
           "ms_per_batch": ms_batch, "wall_ms_per_batch": wall * 1e3 / args.batches,
           "query_signatures_per_sec": Q / (sig_ms * 1e-3),
           "pairs_per_batch": Q * D, "doc_pairs_per_sec": Q * D / (ms_batch * 1e-3),
           "candidates_per_batch": [int(c) for c in cands], "hamming_pairs_per_batch": [int(h) for h in hams],
           "phase_ms_per_batch": {k: v[0] / args.batches for k, v in ph.items() if v[1]},
           "h2d_bytes_per_batch": int(batches[1][0].nbytes)}
    # the two joins alone on the last batch (tiles + scan + emission each)
    for name, fn in (("mrc", lambda: qc.mrc_query_pairs(tau, fetch=False)),
                     ("hamming", lambda: qc.hamming_query_pairs(thr["hamming_max"], fetch=False))):
        qc.set_profiling(True)
        fn()
        p2 = qc.phase_times()
        qc.set_profiling(False)
        tiles, emit = p2["pair_tiles"][0], p2["pair_emit"][0]
        out[name + "_join"] = {"tiles_ms": tiles, "emit_ms": emit, "pairs_per_sec_tiles": Q * D / (tiles * 1e-3),
                               "pairs_per_sec": Q * D / ((tiles + emit) * 1e-3)}
    KP = ((3 * K + 3) + 15) // 16 * 16
    out["mrc_join"]["executed_tflops"] = Q * D * KP * 2 / (out["mrc_join"]["tiles_ms"] * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
