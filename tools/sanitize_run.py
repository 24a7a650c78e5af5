#!/usr/bin/env python3
"""A small pipeline that launches every kernel of librefsig_gpu.so once or
more, under the library's out-of-bounds-write guard:

  REFSIG_CANARY=1 python tools/sanitize_run.py

(every device buffer carries a 4 KB guard region past its end;
Context.debug_check() names any buffer whose guard a kernel overwrote).
compute-sanitizer is closed on the GPU pool this was developed on; the same
script is the memcheck/racecheck/synccheck driver where it is available:

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

K1 (every length class incl. the > 8192-token global path), A5 (reference
docs and explicit vectors, a replaced reference), K2 (lane-per-hit K <= 32,
half-warp short docs, long-doc CTAs, column-owner K = 64 and K = 160), K3 on
tcgen05 (K = 10 one chunk, K = 64 chunked) and on CUDA cores, scan + emit +
keys + csr16, K4a (splitmix and table hashes) and K4b, K5 exact + pair
cosines, the fused evaluation, corpus frequencies and MRCS records, the
query-vs-database join, and the text front end. Checks nothing itself
beyond the library's own validation (the parity tests do that)."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    cp, cfg = C.config_corpus("c0")
    cp = cp.slice_docs(600)
    # lengths across every K1 class edge, plus one > 8192-token document
    rng = np.random.default_rng(5)
    lens = [0, 1, 40, 64, 65, 128, 129, 256, 257, 512, 513, 1024, 1025, 2048, 2049, 4096, 4097, 8192, 9000, 2500]
    extra = [rng.integers(0, cp.vocab, n).astype(np.uint32) for n in lens]
    tok = np.concatenate([cp.tokens] + extra).astype(np.uint32)
    off = np.concatenate([cp.doc_off, cp.doc_off[-1] + np.cumsum(lens)]).astype(np.uint64)
    N = len(off) - 1
    with R.Context(0) as ctx:
        ctx.load_corpus(tok, off, cp.vocab)
        ctx.count(R.WEIGHT_TFIDF)
        ctx.counts()
        ctx.df()
        ctx.corpus_freq()
        ctx.inv_norm()
        for K, path in ((10, R.K3_TENSOR), (10, R.K3_FP32), (64, R.K3_TENSOR), (64, R.K3_FP32), (160, R.K3_AUTO)):
            ctx.set_k3_path(path)
            ctx.set_reference_docs(C.sample_refs(1, N, K))
            ctx.sign()
            ctx.signature_records(7)
            ctx.mrc_pairs(0.9)
            ctx.mrc_pairs_rows(0.5, 128, 384)
            ctx.pairs_csr()
            ctx.pairs_csr16()
            ctx.debug_check()
        ctx.set_k3_path(R.K3_AUTO)
        for K in (129, 200, 224):  # disjoint single-term partitions: the union fills R to its capacity
            ctx.set_reference_partitions([[t] for t in range(K)])
            ctx.sign()
            ctx.debug_check()
        ctx.set_reference_partitions([[1, 2, 3], [4, 5], [7]])
        ctx.sign()
        ctx.mrc_pairs(0.5)
        ctx.simhash(0, R.WEIGHT_TFIDF)
        table = np.arange(cp.vocab, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        ctx.simhash(3, R.WEIGHT_TF, term_hash=table)
        ctx.hamming_pairs(12)
        ctx.exact_pairs(0.5)
        ctx.pair_cosines(np.array([1, (3 << 32) | 9], np.uint64))
        ctx.set_reference_docs(C.sample_refs(2, N, 20))
        ctx.sign(fetch=False)
        ctx.simhash(0)
        ctx.evaluate()
        # the captured step (graph) and its replay
        for _ in range(2):
            ctx.mrc_step(C.sample_refs(3, N, 20), 0.95)
            ctx.step_result(fetch=True)
        ctx.debug_check()
    # query vs database
    with R.Context(0) as db, R.Context(0) as q:
        db.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
        db.count()
        db.set_reference_docs(C.sample_refs(0, cp.n_docs, 128))
        db.sign(fetch=False)
        db.simhash(0)
        q.attach_database(db)
        sub = cp.slice_docs(150)
        q.load_corpus(sub.tokens, sub.doc_off, sub.vocab)
        q.count()
        q.sign(fetch=False)
        q.simhash(0)
        q.mrc_query_pairs(0.9)
        q.hamming_query_pairs(3)
        q.debug_check()
        db.debug_check()
    # text front end
    text, boff = C.synth_text(cp.tokens[: cp.doc_off[200]], cp.doc_off[:201], cp.vocab)
    with R.Context(0) as t:
        t.load_text(text, boff)
        t.count(R.WEIGHT_TF)
        t.counts()
        t.simhash_text()
        t.set_reference_docs(np.arange(5, dtype=np.uint32))
        t.sign(fetch=False)
        t.mrc_pairs(0.9)
        t.debug_check()
    print("sanitize run done: launches", R.Context.launch_count())


if __name__ == "__main__":
    main()
