"""Text front end, CPU: the oracle's restatement of
normalize + extract_3grams + word_hash64 (MD5) + simhash against the golden
fixture made by the reference's own code (tests/golden/text_small.npz), and
live against oracle/_ref on random byte strings when it is built."""
import numpy as np
import pytest

import oracle
from paper_1810_03099_b200 import corpus as C


def grams_entries(text, off):
    tok, goff = oracle.text_grams(text, off)
    return oracle.count(tok, goff)


def test_text_grams_vs_reference_fixture(golden_text):
    g = golden_text
    c = grams_entries(g["text"], g["byte_off"])
    assert np.array_equal(c.rowptr, g["rowptr"])
    assert np.array_equal(c.ids, g["ids"])
    assert np.array_equal(c.counts, g["counts"])


def test_text_simhash_vs_reference_fixture(golden_text):
    g = golden_text
    assert np.array_equal(oracle.text_simhash(g["text"], g["byte_off"]), g["fp"])


def test_word_hash64_padding_edges(golden_text):
    g = golden_text
    for w, h in zip(g["words"], g["word_hash"]):
        assert oracle.word_hash64(str(w).encode()) == int(h), w


R = oracle.ref_lib()


@pytest.mark.skipif(R is None, reason="oracle/_ref not built (make ref)")
@pytest.mark.parametrize("seed", range(4))
def test_text_front_end_vs_reference_live(seed):
    import ctypes
    rng = np.random.default_rng(seed)
    alphabet = np.frombuffer(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ  .,;-'0123456789\n\xc3\xa9\xff", np.uint8)
    docs = [bytes(alphabet[rng.integers(0, len(alphabet), rng.integers(0, 400))]) for _ in range(40)]
    text = np.frombuffer(b"".join(docs) or b"\0", np.uint8)
    off = np.zeros(len(docs) + 1, np.uint64)
    np.cumsum([len(x) for x in docs], out=off[1:])
    c = grams_entries(text, off)
    fp = oracle.text_simhash(text, off)
    U32 = ctypes.POINTER(ctypes.c_uint32)
    for d, x in enumerate(docs):
        cap = len(x) + 8
        oi = np.empty(cap, np.uint32)
        oc = np.empty(cap, np.uint32)
        k = R.ref_extract_3grams(x, len(x), oi.ctypes.data_as(U32), oc.ctypes.data_as(U32), cap)
        lo, hi = int(c.rowptr[d]), int(c.rowptr[d + 1])
        assert np.array_equal(c.ids[lo:hi], oi[:k]) and np.array_equal(c.counts[lo:hi], oc[:k])
        nb = ctypes.create_string_buffer(len(x) + 1)
        m = R.ref_normalize(x, len(x), nb, len(x) + 1)
        words = [w for w in nb.raw[:m].split(b" ") if w]
        packed = b"".join(words)
        lens = np.array([len(w) for w in words] or [0], np.uint64)
        ref = R.ref_simhash(packed, lens.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(words))
        assert int(fp[d]) == int(ref)


def test_synth_text_is_deterministic():
    cp, _ = C.config_corpus("c0")
    cp = cp.slice_docs(50)
    a = C.synth_text(cp.tokens, cp.doc_off, cp.vocab, seed=3)
    b = C.synth_text(cp.tokens, cp.doc_off, cp.vocab, seed=3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
