"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
golden fixtures made from the reference's own code.

Bars (north_star / SURVEY.md §8c): counts, df, idf32, Simhash fingerprints
and Hamming pairs bit-exact; signatures |g-c| <= 1e-5*|c| + 1e-7; candidate
pair sets identical except pairs whose oracle score is within 1e-5 of the
threshold (listed by the oracle and reported here)."""
import numpy as np
import pytest

import oracle
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C

pytestmark = pytest.mark.gpu

SIG_RTOL, SIG_ATOL = 1e-5, 1e-7
BAND = 1e-5


def assert_sig_close(g, c):
    err = np.abs(g.astype(np.float64) - c)
    bad = err > SIG_RTOL * np.abs(c) + SIG_ATOL
    assert not bad.any(), f"{bad.sum()} signature values out of tolerance, max err {err.max():.3g}"


from tests.parity_util import assert_pairs_match  # noqa: E402  (numpy set algebra, border rule)


def corpus_c0(n=None):
    cp, cfg = C.config_corpus("c0")
    if n:
        cp = cp.slice_docs(n)
    return cp, cfg


def gpu_pipeline(ctx, cp, refs, weighting=R.WEIGHT_TFIDF):
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count(weighting)
    ctx.set_reference_docs(refs)
    return ctx.sign()


def oracle_pipeline(cp, refs, weighting="tfidf"):
    return oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs, weighting)


# ---- K1 -------------------------------------------------------------------

def test_counts_match_reference_golden(gpu_ctx_factory, golden_small):
    g = golden_small
    ctx = gpu_ctx_factory()
    ctx.load_corpus(g["tokens"], g["doc_off"], int(g["vocab"]))
    ctx.count(R.WEIGHT_TF)
    rowptr, ids, counts = ctx.counts()
    # includes an empty doc, a single-term doc and a 9000-token doc (global-scratch path)
    assert np.array_equal(rowptr, g["rowptr"])
    assert np.array_equal(ids, g["ids"])
    assert np.array_equal(counts, g["counts"])


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_counts_df_idf_bitexact(gpu_ctx_factory, name):
    cp, cfg = C.config_corpus(name)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count(R.WEIGHT_TFIDF)
    rowptr, ids, counts = ctx.counts()
    c = oracle.count(cp.tokens, cp.doc_off)
    assert np.array_equal(rowptr, c.rowptr)
    assert np.array_equal(ids, c.ids)
    assert np.array_equal(counts, c.counts)
    df, idf = ctx.df()
    odf = oracle.df(c, cp.vocab)
    assert np.array_equal(df, odf)
    assert np.array_equal(idf.view(np.uint32), oracle.idf32(odf, cp.n_docs).view(np.uint32))


def test_count_length_bins_and_long_docs(gpu_ctx_factory):
    # lengths straddling every bin edge (256/1024/4096/8192) and > 8192
    rng = np.random.default_rng(3)
    lens = [0, 1, 255, 256, 257, 1023, 1024, 1025, 4095, 4096, 4097, 8191, 8192, 8193, 20000, 3, 70000]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    V = 1000
    tok = rng.integers(0, V, int(off[-1]), dtype=np.uint32)
    tok[off[2]:off[3]] = 7  # one doc of a single repeated term
    ctx = gpu_ctx_factory()
    ctx.load_corpus(tok, off, V)
    ctx.count(R.WEIGHT_TF)
    rowptr, ids, counts = ctx.counts()
    c = oracle.count(tok, off)
    assert np.array_equal(rowptr, c.rowptr) and np.array_equal(ids, c.ids) and np.array_equal(counts, c.counts)


# ---- K2 -------------------------------------------------------------------

def test_sign_partitions_match_reference_golden(gpu_ctx_factory, golden_small):
    g = golden_small
    ctx = gpu_ctx_factory()
    ctx.load_corpus(g["tokens"], g["doc_off"], int(g["vocab"]))
    ctx.count(R.WEIGHT_TF)
    ctx.set_reference_vectors(g["part_rowptr"], g["part_ids"])
    S = ctx.sign()
    assert_sig_close(S, g["sig_tf"])


@pytest.mark.parametrize("K", [1, 7, 10, 16, 20, 23, 27, 32, 64, 128, 160])  # every K <= 32 column-group width
def test_sign_c0_vs_oracle(gpu_ctx_factory, K):
    cp, cfg = corpus_c0()
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, K)
    ctx = gpu_ctx_factory()
    S = gpu_pipeline(ctx, cp, refs)
    o = oracle_pipeline(cp, refs)
    assert_sig_close(S, o.S)
    # self-similarity: a reference doc's own column is 1
    for k, d in enumerate(refs[:8]):
        assert abs(S[d, k] - 1.0) <= 1e-6


def test_sign_c1_vs_oracle(gpu_ctx_factory):
    cp, cfg = C.config_corpus("c1")
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = gpu_ctx_factory()
    S = gpu_pipeline(ctx, cp, refs)
    o = oracle_pipeline(cp, refs)
    assert_sig_close(S, o.S)


def test_disjoint_doc_gives_zero_signature(gpu_ctx_factory):
    # docs sharing no term with any reference sign to all-zero
    tok = np.array([1, 2, 3, 1, 4, 5, 6, 100, 101], np.uint32)
    off = np.array([0, 4, 7, 9], np.uint64)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(tok, off, 200)
    ctx.count(R.WEIGHT_TF)
    ctx.set_reference_partitions([[1, 2], [3]])
    S = ctx.sign()
    assert np.all(S[1] == 0) and np.all(S[2] == 0)
    assert S[0, 0] > 0 and S[0, 1] > 0
    # all-zero signatures compare as 0: never >= tau > 0
    assert len(ctx.mrc_pairs(1e-9)) == 0
    # ... and as 0 >= tau for tau <= 0, like the reference's compare
    assert len(ctx.mrc_pairs(0.0)) == 3


# ---- K3 -------------------------------------------------------------------

@pytest.mark.parametrize("tau", [0.5, 0.9, 0.99, 0.999])
def test_mrc_pairs_c0_vs_oracle(gpu_ctx_factory, tau):
    cp, cfg = corpus_c0()
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = gpu_ctx_factory()
    gpu_pipeline(ctx, cp, refs)
    keys = ctx.mrc_pairs(tau)
    o = oracle_pipeline(cp, refs)
    pairs, border = oracle.mrc_pairs(o.S, tau, BAND)
    assert_pairs_match(keys, pairs, border, f"tau={tau}")


@pytest.mark.parametrize("K", [1, 2, 7, 41, 42])
def test_mrc_pairs_tensor_core_k_edges(gpu_ctx_factory, K):
    """K3 runs on tcgen05 for 3K + 3 <= 128 (K <= 41) and on FP32 CUDA cores
    above: both sides of the switch, and the smallest K'."""
    cp, cfg = corpus_c0(1500)
    refs = C.sample_refs(7, cp.n_docs, K)
    ctx = gpu_ctx_factory()
    gpu_pipeline(ctx, cp, refs)
    o = oracle_pipeline(cp, refs)
    for tau in (0.5, 0.9):
        keys = ctx.mrc_pairs(tau)
        pairs, border = oracle.mrc_pairs(o.S, tau, BAND)
        assert_pairs_match(keys, pairs, border, f"K={K} tau={tau}")


def test_mrc_pairs_c1_vs_oracle(gpu_ctx_factory):
    cp, cfg = C.config_corpus("c1")
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = gpu_ctx_factory()
    gpu_pipeline(ctx, cp, refs)
    tau = C.load_configs()["thresholds"]["tau_mrc"]
    keys = ctx.mrc_pairs(tau)
    o = oracle_pipeline(cp, refs)
    pairs, border = oracle.mrc_pairs(o.S, tau, BAND)
    nb = assert_pairs_match(keys, pairs, border, "c1")
    print(f"c1 tau={tau}: {len(keys)} GPU pairs, {len(pairs)} oracle pairs, {len(border)} in band, {nb} differ")


def test_mrc_pairs_overflow_reports_exact_count(gpu_ctx_factory):
    cp, cfg = corpus_c0(500)
    refs = C.sample_refs(0, cp.n_docs, 10)
    ctx = gpu_ctx_factory()
    gpu_pipeline(ctx, cp, refs)
    full = ctx.mrc_pairs(0.9)
    assert len(full) > 10
    buf = np.zeros(10, np.uint64)
    with pytest.raises(R.PairOverflowError) as e:
        ctx.mrc_pairs(0.9, out=buf)
    assert e.value.count == len(full)
    assert np.array_equal(buf, full[:10])


def test_duplicate_docs_match(gpu_ctx_factory):
    cp, _ = corpus_c0(300)
    # append exact copies of docs 3 and 7
    extra = [cp.tokens[cp.doc_off[d]:cp.doc_off[d + 1]] for d in (3, 7)]
    tok = np.concatenate([cp.tokens] + extra)
    off = np.concatenate([cp.doc_off, cp.doc_off[-1] + np.cumsum([len(x) for x in extra])]).astype(np.uint64)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(tok, off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(C.sample_refs(0, 300, 10))
    ctx.sign(fetch=False)
    keys = set(ctx.mrc_pairs(0.99999).tolist())
    assert (3 << 32 | 300) in keys and (7 << 32 | 301) in keys
    ex = set(ctx.exact_pairs(0.99999).tolist())
    assert (3 << 32 | 300) in ex and (7 << 32 | 301) in ex


# ---- K4 -------------------------------------------------------------------

def test_simhash_md5_table_matches_reference_golden(gpu_ctx_factory, golden_small):
    g = golden_small
    ctx = gpu_ctx_factory()
    ctx.load_corpus(g["tokens"], g["doc_off"], int(g["vocab"]))
    ctx.count(R.WEIGHT_TF)
    fp = ctx.simhash(0, R.WEIGHT_TF, term_hash=g["term_hash"])
    assert np.array_equal(fp, g["fp_md5"])  # refsig::simhash over MD5 words, bit-exact


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_simhash_tfidf_bitexact(gpu_ctx_factory, name):
    cp, cfg = C.config_corpus(name)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count(R.WEIGHT_TFIDF)
    fp = ctx.simhash(0, R.WEIGHT_TFIDF)
    c = oracle.count(cp.tokens, cp.doc_off)
    ofp = oracle.simhash(c, oracle.idf32(oracle.df(c, cp.vocab), cp.n_docs), seed=0)
    assert np.array_equal(fp, ofp)
    fp_tf = ctx.simhash(7, R.WEIGHT_TF)
    assert np.array_equal(fp_tf, oracle.simhash(c, None, seed=7))


@pytest.mark.parametrize("max_dist", [0, 3, 12])
def test_hamming_pairs_bitexact(gpu_ctx_factory, max_dist):
    cp, cfg = C.config_corpus("c1")
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    fp = ctx.simhash(0)
    keys = ctx.hamming_pairs(max_dist)
    want = oracle.hamming_pairs(fp, max_dist)
    assert np.array_equal(keys, want)


# ---- K5 -------------------------------------------------------------------

@pytest.mark.parametrize("tau", [0.3, 0.8])
def test_exact_pairs_c0_vs_oracle(gpu_ctx_factory, tau):
    cp, cfg = corpus_c0()
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    keys = ctx.exact_pairs(tau)
    o = oracle_pipeline(cp, C.sample_refs(0, cp.n_docs, 10))
    pairs, border = oracle.exact_pairs(o.x, cp.vocab, tau, BAND)
    assert_pairs_match(keys, pairs, border, f"exact tau={tau}")


def test_exact_pairs_c1_rows_vs_oracle(gpu_ctx_factory):
    cp, cfg = C.config_corpus("c1")
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    tau = C.load_configs()["thresholds"]["tau_cos"]
    keys = ctx.exact_pairs(tau)
    o = oracle_pipeline(cp, C.sample_refs(0, cp.n_docs, 20))
    rows = 2000  # oracle panel: rows [0, 2000) x all j > i
    pairs, border = oracle.exact_pairs(o.x, cp.vocab, tau, BAND, 0, rows)
    gk = keys[(keys >> np.uint64(32)) < rows]
    assert_pairs_match(gk, pairs, border, "exact c1 rows")
    # planted near-duplicates (10% resampled) are found
    dups = np.nonzero(cp.dup_src != 0xFFFFFFFF)[0]
    ks = set(keys.tolist())
    found = sum(((min(d, int(cp.dup_src[d])) << 32) | max(d, int(cp.dup_src[d]))) in ks for d in dups)
    assert found / len(dups) > 0.5


def test_pair_cosines_match_reference_golden(gpu_ctx_factory, golden_small):
    g = golden_small
    ctx = gpu_ctx_factory()
    ctx.load_corpus(g["tokens"], g["doc_off"], int(g["vocab"]))
    ctx.count(R.WEIGHT_TF)
    cos = ctx.pair_cosines(g["pair_keys"])
    np.testing.assert_allclose(cos, g["pair_cos"], rtol=1e-5, atol=1e-7)


# ---- errors (reference error.hpp:8-14 mapping) ----------------------------

@pytest.mark.parametrize("length", [3, 100, 200, 400, 1000, 3000, 6000, 12000])
def test_out_of_vocab_id_every_count_class(gpu_ctx_factory, length):
    """An id >= vocab is reported (ValidationError) by every K1 work class
    (warp sorts, CTA sorts, the global-memory path), wherever it sits."""
    rng = np.random.default_rng(length)
    for pos in (0, length - 1):
        tok = rng.integers(0, 1000, length).astype(np.uint32)
        tok[pos] = 1000
        ctx = gpu_ctx_factory()
        ctx.load_corpus(np.r_[tok, tok].astype(np.uint32), np.array([0, length, 2 * length], np.uint64), 1000)
        ctx.count()
        with pytest.raises(R.ValidationError, match="vocab"):
            ctx.synchronize()


def test_validation_errors(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    with pytest.raises(R.ValidationError):
        ctx.count()  # no corpus
    with pytest.raises(R.ValidationError):
        ctx.load_corpus(np.zeros(0, np.uint32), np.array([0], np.uint64), 10)  # empty corpus
    tok = np.array([1, 2, 50], np.uint32)
    ctx.load_corpus(tok, np.array([0, 3], np.uint64), 10)  # id 50 >= vocab 10
    ctx.count()
    with pytest.raises(R.ValidationError, match="vocab"):
        ctx.synchronize()
    ctx.load_corpus(np.array([1, 2], np.uint32), np.array([0, 2], np.uint64), 10)
    ctx.count()
    with pytest.raises(R.ValidationError):
        ctx.set_reference_docs([])
    with pytest.raises(R.ValidationError):
        ctx.set_reference_docs([5])  # >= n_docs
    with pytest.raises(R.ValidationError, match="1..256"):
        ctx.set_reference_docs(np.zeros(257, np.uint32))  # K above the K2 register budget
    with pytest.raises(R.ValidationError):
        ctx.mrc_pairs(0.9)  # not signed
    with pytest.raises(R.ValidationError):
        ctx.set_reference_vectors([0, 2], [3, 3])  # duplicate term
    with pytest.raises(R.ValidationError):
        ctx.hamming_pairs(3)  # no fingerprints


def test_query_vs_database(gpu_ctx_factory):
    cfg = C.load_configs()["configs"]["c4"]
    db_spec = dict(cfg["corpus"], n_docs=4000, vocab=50000)
    q_spec = dict(cfg["queries"], n_docs=600, vocab=50000)
    db = C.generate(db_spec)
    q = C.generate_queries(q_spec, db_spec, db)
    K = 32
    refs = C.sample_refs(0, db.n_docs, K)
    dbc = gpu_ctx_factory()
    dbc.load_corpus(db.tokens, db.doc_off, db.vocab)
    dbc.count()
    dbc.set_reference_docs(refs)
    Sd = dbc.sign()
    fd = dbc.simhash(0)
    qc = gpu_ctx_factory()
    qc.attach_database(dbc)
    qc.load_corpus(q.tokens, q.doc_off, q.vocab)
    qc.count()
    Sq = qc.sign()
    fq = qc.simhash(0)
    # oracle: queries weighted with the database IDF, signed against its refs
    od = oracle.mrc_pipeline(db.tokens, db.doc_off, db.vocab, refs)
    cq = oracle.count(q.tokens, q.doc_off)
    xq = oracle.weighted(cq, od.idf)
    oSq = oracle.sign(xq, oracle.rows(od.x, refs))
    assert_sig_close(Sd, od.S)
    assert_sig_close(Sq, oSq)
    keys = qc.mrc_query_pairs(0.99)
    pairs, border = oracle.mrc_query_pairs(oSq, od.S, 0.99, BAND)
    assert_pairs_match(keys, pairs, border, "query mrc")
    hk = qc.hamming_query_pairs(3)
    assert np.array_equal(hk, oracle.hamming_query_pairs(oracle.simhash(cq, od.idf, 0), fd, 3))
    assert np.array_equal(fq, oracle.simhash(cq, od.idf, 0))


def test_reference_replaced_and_union(gpu_ctx_factory):
    # a second reference on the same counts must not see the first one's rows
    cp, cfg = corpus_c0(800)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    r1 = C.sample_refs(1, cp.n_docs, 10)
    r2 = C.sample_refs(2, cp.n_docs, 7)
    ctx.set_reference_docs(r1)
    ctx.sign(fetch=False)
    ctx.set_reference_docs(r2)
    S2 = ctx.sign()
    o = oracle_pipeline(cp, r2)
    assert_sig_close(S2, o.S)
    c = o.counts
    union = set()
    for d in r2:
        union.update(c.ids[c.rowptr[d]:c.rowptr[d + 1]].tolist())
    assert ctx.reference_union() == len(union)
    # explicit vectors after doc references
    ctx.set_reference_partitions([[1, 2, 3], [4, 5]])
    S3 = ctx.sign()
    ref = oracle.vectors([0, 3, 5], [1, 2, 3, 4, 5], np.ones(5))
    assert_sig_close(S3, oracle.sign(o.x, ref))


def test_pairs_csr_matches_keys(gpu_ctx_factory):
    """get_pairs_csr is the same sorted pair list as the 64-bit keys."""
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(5000)
    refs = C.sample_refs(0, cp.n_docs, 20)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(refs)
    ctx.sign(fetch=False)
    keys = ctx.mrc_pairs(0.95)
    rowptr, cols = ctx.pairs_csr()
    assert rowptr[0] == 0 and rowptr[-1] == len(keys) == len(cols)
    rows = np.repeat(np.arange(cp.n_docs, dtype=np.uint64), np.diff(rowptr).astype(np.int64))
    assert np.array_equal((rows << np.uint64(32)) | cols.astype(np.uint64), keys)
    # a row slice, caller buffers, and overflow reporting
    rp, cs = ctx.pairs_csr(128, 1024)
    lo, hi = np.searchsorted(keys >> np.uint64(32), [128, 1024])
    assert np.array_equal(cs, (keys[lo:hi] & np.uint64(0xFFFFFFFF)).astype(np.uint32))
    assert np.array_equal(rp, np.searchsorted(keys[lo:hi] >> np.uint64(32), np.arange(128, 1025)))
    if len(keys) > 1:
        with pytest.raises(R.PairOverflowError):
            ctx.pairs_csr(cols=np.empty(len(keys) - 1, np.uint32))


@pytest.mark.parametrize("weighting", [R.WEIGHT_TF, R.WEIGHT_TFIDF])
def test_evaluate_vs_oracle(gpu_ctx_factory, weighting):
    """SPEC eval (Eq. 2/3) fused on the GPU: MAE, mean error and variance of MRC
    and Simhash against the exact cosine over all pairs (c0 shape, 1200 docs)."""
    cp, cfg = C.config_corpus("c0")
    cp = cp.slice_docs(1200)
    refs = C.sample_refs(0, cp.n_docs, cfg["K"])
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count(weighting)
    ctx.set_reference_docs(refs)
    ctx.sign(fetch=False)
    ctx.simhash(0, weighting)
    g = ctx.evaluate()
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs,
                            "tfidf" if weighting == R.WEIGHT_TFIDF else "tf")
    fp = oracle.simhash(o.counts, o.idf if weighting == R.WEIGHT_TFIDF else None, 0)
    ref = oracle.evaluate(o.x, o.S, fp)
    assert g["pairs"] == ref["pairs"] == cp.n_docs * (cp.n_docs - 1) // 2
    for k in ("mrc_mae", "mrc_mean_error", "simhash_mae", "simhash_mean_error"):
        assert abs(g[k] - ref[k]) <= 2e-6 + 1e-5 * abs(ref[k]), (k, g[k], ref[k])
    for k in ("mrc_variance", "simhash_variance"):
        assert abs(g[k] - ref[k]) <= 1e-7 + 1e-4 * abs(ref[k]), (k, g[k], ref[k])
    # a row range (two 128-row panels) matches the oracle's same range
    g2 = ctx.evaluate(128, 384)
    ref2 = oracle.evaluate(o.x, o.S, fp, 128, 384)
    assert g2["pairs"] == ref2["pairs"]
    assert abs(g2["mrc_mae"] - ref2["mrc_mae"]) <= 2e-6 + 1e-5 * abs(ref2["mrc_mae"])


def test_pairs_csr16_matches_csr32(gpu_ctx_factory):
    cp, cfg = corpus_c0()
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = gpu_ctx_factory()
    gpu_pipeline(ctx, cp, refs)
    ctx.mrc_pairs(0.9, fetch=False)
    rp32, c32 = ctx.pairs_csr()
    rp16, c16 = ctx.pairs_csr16()
    assert c16.dtype == np.uint16 and np.array_equal(rp16, rp32) and np.array_equal(c16.astype(np.uint32), c32)
    rp, c = ctx.pairs_csr16(128, 640)  # a row range, rowptr rebased to 0
    r32, c3 = ctx.pairs_csr(128, 640)
    assert np.array_equal(rp, r32) and np.array_equal(c.astype(np.uint32), c3)
    # more than 65536 columns: 16-bit ids refused
    n = 70000
    big = gpu_ctx_factory()
    big.load_corpus(np.arange(n, dtype=np.uint32) % 50, np.arange(n + 1, dtype=np.uint64), 50)
    big.count(R.WEIGHT_TF)
    big.set_reference_docs(np.arange(4, dtype=np.uint32))
    big.sign(fetch=False)
    big.mrc_pairs(2.0, fetch=False)
    with pytest.raises(R.ValidationError, match="65536"):
        big.pairs_csr16()
