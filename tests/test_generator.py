"""Synthetic corpus generator (input stand-in for NEWS20). CPU only."""
import numpy as np

from paper_1810_03099_b200 import corpus as C


def test_deterministic_and_thread_invariant():
    spec = C.load_configs()["configs"]["c1"]["corpus"].copy()
    spec["n_docs"] = 1500
    a = C.generate(spec, threads=1)
    b = C.generate(spec, threads=7)
    assert np.array_equal(a.doc_off, b.doc_off)
    assert np.array_equal(a.tokens, b.tokens)
    assert np.array_equal(a.dup_src, b.dup_src)


def test_c0_shape():
    cp, cfg = C.config_corpus("c0")
    L = np.diff(cp.doc_off.astype(np.int64))
    assert cp.n_docs == 2000
    assert L.min() >= 10 and L.max() <= 5000
    assert 130 <= np.median(L) <= 170  # lognormal median 150
    assert cp.tokens.max() < 30000
    assert np.all(cp.dup_src == 0xFFFFFFFF)
    # Zipf: rank 0 is the most frequent term of the global distribution
    f = np.bincount(cp.tokens, minlength=30000)
    assert f.argmax() == 0


def test_c1_near_duplicates():
    cp, cfg = C.config_corpus("c1")
    assert cp.n_docs == 18846
    dups = np.nonzero(cp.dup_src != 0xFFFFFFFF)[0]
    assert len(dups) == round(0.05 * 18846)
    # a near-dup copies its (original) source's length and ~90% of its tokens
    for d in dups[:50]:
        s = int(cp.dup_src[d])
        assert cp.dup_src[s] == 0xFFFFFFFF
        a = cp.tokens[cp.doc_off[d]:cp.doc_off[d + 1]]
        b = cp.tokens[cp.doc_off[s]:cp.doc_off[s + 1]]
        assert len(a) == len(b)
        if len(a) >= 100:
            assert 0.75 < np.mean(a == b) < 0.97


def test_reference_sampling():
    r = C.sample_refs(0, 18846, 20)
    assert len(set(r.tolist())) == 20 and r.max() < 18846
    assert np.array_equal(r, C.sample_refs(0, 18846, 20))
    r2 = C.sample_refs(0, 1_000_000, 128)
    assert len(set(r2.tolist())) == 128


def test_query_batch_near_dups_of_db():
    cfg = C.load_configs()["configs"]["c4"]
    db_spec = dict(cfg["corpus"], n_docs=3000)
    q_spec = dict(cfg["queries"], n_docs=500)
    db = C.generate(db_spec)
    q = C.generate_queries(q_spec, db_spec, db)
    src = q.dup_src
    dups = np.nonzero(src != 0xFFFFFFFF)[0]
    assert len(dups) == 50
    assert src[dups].max() < 3000
