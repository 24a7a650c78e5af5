"""GPU text front end against the reference's own
outputs (tests/golden/text_small.npz, made by refsig::extract_3grams /
refsig::simhash) and the oracle at larger sizes; then the whole MRC path on
the 3-gram corpus it produces."""
import numpy as np
import pytest

import oracle
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
from tests.test_gpu_parity import BAND, assert_pairs_match

pytestmark = pytest.mark.gpu


def test_text_grams_and_simhash_vs_reference(gpu_ctx_factory, golden_text):
    g = golden_text
    ctx = gpu_ctx_factory()
    ctx.load_text(g["text"], g["byte_off"])
    assert ctx.vocab == 17576
    ctx.count(R.WEIGHT_TF)
    rowptr, ids, counts = ctx.counts()
    assert np.array_equal(rowptr, g["rowptr"])
    assert np.array_equal(ids, g["ids"])
    assert np.array_equal(counts, g["counts"])
    assert np.array_equal(ctx.simhash_text(), g["fp"])  # refsig::simhash over MD5 words, bit-exact


def test_text_front_end_c1_vs_oracle(gpu_ctx_factory):
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(4000)
    text, off = C.synth_text(cp.tokens, cp.doc_off, cp.vocab, seed=1)
    tok, goff = oracle.text_grams(text, off)
    ctx = gpu_ctx_factory()
    ctx.load_text(text, off)
    ctx.count(R.WEIGHT_TFIDF)
    c = oracle.count(tok, goff)
    rowptr, ids, counts = ctx.counts()
    assert np.array_equal(rowptr, c.rowptr) and np.array_equal(ids, c.ids) and np.array_equal(counts, c.counts)
    assert np.array_equal(ctx.simhash_text(), oracle.text_simhash(text, off))
    # the MRC path on the 3-gram corpus
    refs = C.sample_refs(0, cp.n_docs, 20)
    ctx.set_reference_docs(refs)
    S = ctx.sign()
    o = oracle.mrc_pipeline(tok, goff, 17576, refs)
    np.testing.assert_allclose(S, o.S, rtol=1e-5, atol=1e-7)
    keys = ctx.mrc_pairs(0.999)
    pairs, border = oracle.mrc_pairs(o.S, 0.999, BAND)
    assert_pairs_match(keys, pairs, border, "text mrc")


def test_text_reload_and_empty(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    ctx.load_text(b"", np.array([0, 0], np.uint64))  # one empty doc
    ctx.count(R.WEIGHT_TF)
    assert ctx.counts()[0].tolist() == [0, 0]
    assert ctx.simhash_text().tolist() == [0]
    ctx.load_text(b"abcd ABCD", np.array([0, 4, 9], np.uint64))
    ctx.count(R.WEIGHT_TF)
    rowptr, ids, counts = ctx.counts()
    assert rowptr.tolist() == [0, 2, 4] and ids.tolist() == [28, 731] * 2 and counts.tolist() == [1, 1, 1, 1]
    a = ctx.simhash_text()
    assert a[0] == a[1] == oracle.word_hash64(b"abcd")  # one word: its hash
    with pytest.raises(R.ValidationError):
        ctx.load_text(b"ab", np.array([0, 3], np.uint64))  # offsets beyond the text are the caller's bug
