"""f4 on the GPU: corpus_freq / doc_freq reductions behind the frequency table,
the device-written MRCS records, and a Reference (MRCREF) driving sign().
Known answers: SPEC.md:219-221, the reference's own extract_3grams output
(tests/golden/text_small.npz) and bincount over the token stream at
configs[1] size."""
import numpy as np
import pytest

import oracle
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
from paper_1810_03099_b200 import formats as F

pytestmark = pytest.mark.gpu


def load_docs(ctx, docs):
    text = b"".join(d.encode() for d in docs)
    off = np.r_[0, np.cumsum([len(d) for d in docs])].astype(np.uint64)
    ctx.load_text(text, off)
    ctx.count(R.WEIGHT_TF)
    return text, off


def test_frequency_table_spec_examples_gpu(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    load_docs(ctx, ["abcd", "abcx"])
    assert F.build_frequency_table(ctx).rows() == [("abc", 2, 2), ("bcd", 1, 1), ("bcx", 1, 1)]
    load_docs(ctx, ["aaaa"])
    assert F.build_frequency_table(ctx).rows() == [("aaa", 2, 1)]
    load_docs(ctx, ["ab cd", "", "x"])
    assert len(F.build_frequency_table(ctx)) == 0


def test_frequency_table_vs_reference_golden(gpu_ctx_factory, golden_text):
    g = golden_text
    ctx = gpu_ctx_factory()
    ctx.load_text(g["text"], g["byte_off"])
    ctx.count(R.WEIGHT_TFIDF)
    # cf/df from the reference's own per-doc NgramVectors (refsig::extract_3grams)
    cf = np.bincount(g["ids"], weights=g["counts"], minlength=F.GRAM_SPACE).astype(np.uint64)
    df = np.bincount(g["ids"], minlength=F.GRAM_SPACE).astype(np.uint64)
    assert np.array_equal(ctx.corpus_freq(), cf)
    assert F.build_frequency_table(ctx) == F.FrequencyTable.from_counts(cf, df)


def test_corpus_freq_full_size(gpu_ctx_factory):
    cp, _ = C.config_corpus("c1")
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count(R.WEIGHT_TFIDF)
    cf = ctx.corpus_freq()
    assert np.array_equal(cf, np.bincount(cp.tokens, minlength=cp.vocab).astype(np.uint64))
    assert int(cf.sum()) == len(cp.tokens)
    d, _ = ctx.df()
    assert np.all(cf >= d) and np.array_equal(cf > 0, d > 0)


def test_text_to_table_to_reference_to_mrcs(gpu_ctx_factory, tmp_path):
    cp, _ = C.config_corpus("c1")
    cp = cp.slice_docs(3000)
    text, off = C.synth_text(cp.tokens, cp.doc_off, cp.vocab, seed=4)
    ctx = gpu_ctx_factory()
    ctx.load_text(text, off)
    ctx.count(R.WEIGHT_TF)  # SPEC sign(): cosine of raw-count NgramVectors
    t = F.build_frequency_table(ctx)
    F.save_frequency_table(t, tmp_path / "t.tsv")
    t = F.load_frequency_table(tmp_path / "t.tsv")
    for gl, P in [(F.build_band(t, 0, 600), 30), (F.build_infogain(t, 1500), 60), (F.build_nonzero(t), 40)]:
        ref = F.partition(gl, P)
        F.save_reference(ref, tmp_path / "r.ref")
        ref = F.load_reference(tmp_path / "r.ref")
        ref.install(ctx)
        S = ctx.sign()
        # oracle: sign against the same count-1 partition vectors
        tok, goff = oracle.text_grams(text, off)
        c = oracle.count(tok, goff)
        x = oracle.weighted(c, None)
        refv = oracle.vectors(ref.rowptr, np.asarray(ref.grams.grams, np.uint32), np.ones(ref.L, np.float32))
        S_or = oracle.sign(x, refv)
        np.testing.assert_allclose(S, S_or, rtol=1e-5, atol=1e-7)
        rid = ref.ref_id
        rec = ctx.signature_records(rid)
        assert rec.shape == (len(off) - 1, 20 + 8 * P)
        S64, ids = F.decode_records(rec)
        assert np.all(ids == rid)
        assert S64.tobytes() == S.astype(np.float64).tobytes()  # exact widening
        F.write_signature_files(tmp_path / "sig", [f"{d}.mrcs" for d in range(3)], rec[:3])
        v, r1 = F.load_signature(tmp_path / "sig" / "1.mrcs")
        assert r1 == rid and v.tobytes() == S[1].astype(np.float64).tobytes()


@pytest.mark.parametrize("K", [1, 7, 32, 33, 256])
def test_signature_records_all_K(gpu_ctx_factory, golden_small, K):
    g = golden_small
    ctx = gpu_ctx_factory()
    ctx.load_corpus(g["tokens"], g["doc_off"], int(g["vocab"]))
    ctx.count(R.WEIGHT_TFIDF)
    n = len(g["doc_off"]) - 1
    ctx.set_reference_docs(np.arange(K, dtype=np.uint32) % n)
    S = ctx.sign()
    rec = ctx.signature_records(0xFEEDFACECAFEBEEF)
    assert rec.shape == (n, 20 + 8 * K)
    assert bytes(rec[0, :4]) == b"MRCS"
    S64, ids = F.decode_records(rec)
    assert np.all(ids == 0xFEEDFACECAFEBEEF) and S64.tobytes() == S.astype(np.float64).tobytes()
    with pytest.raises(R.ValidationError):
        ctx._check(ctx._L.refsig_gpu_get_signature_records(ctx._h, 1, R._ptr(rec, __import__("ctypes").c_uint8), 8))
