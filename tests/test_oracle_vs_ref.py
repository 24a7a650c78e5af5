"""Pin the oracle restatement against the reference's own code, live
(oracle/_ref/librefshim.so compiled from the reference headers), on random
inputs beyond the committed golden fixtures. CPU only."""
import ctypes

import numpy as np
import pytest

import oracle

R = oracle.ref_lib()
pytestmark = pytest.mark.skipif(R is None, reason="oracle/_ref not built (make ref)")
U32 = ctypes.POINTER(ctypes.c_uint32)


def ref_entries(ids):
    ids = np.ascontiguousarray(ids, np.uint32)
    n = len(ids)
    oi = np.empty(max(n, 1), np.uint32)
    oc = np.empty(max(n, 1), np.uint32)
    k = R.ref_from_entries(ids.ctypes.data_as(U32), None, n, oi.ctypes.data_as(U32), oc.ctypes.data_as(U32), None)
    return oi[:k], oc[:k]


@pytest.mark.parametrize("seed", range(5))
def test_counts_equal_from_entries(seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 400, 60)
    lens[0] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    vocab = int(rng.integers(5, 50000))
    tok = rng.integers(0, vocab, int(off[-1]), dtype=np.uint32)
    c = oracle.count(tok, off, threads=3)
    for d in range(len(lens)):
        i, n = ref_entries(tok[off[d]:off[d + 1]])
        b, e = int(c.rowptr[d]), int(c.rowptr[d + 1])
        assert np.array_equal(c.ids[b:e], i) and np.array_equal(c.counts[b:e], n)


@pytest.mark.parametrize("seed", range(3))
def test_tf_cosine_equals_reference_cosine(seed):
    rng = np.random.default_rng(100 + seed)
    lens = rng.integers(0, 120, 40)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    tok = rng.integers(0, 60, int(off[-1]), dtype=np.uint32)  # small vocab: many overlaps
    c = oracle.count(tok, off, threads=1)
    x = oracle.weighted(c, None)
    iu = np.triu_indices(len(lens), 1)
    keys = (iu[0].astype(np.uint64) << np.uint64(32)) | iu[1].astype(np.uint64)
    got = oracle.cosine_pairs(x, keys, threads=2)
    for q in range(0, len(keys), 7):
        i, j = int(iu[0][q]), int(iu[1][q])
        a = c.ids[c.rowptr[i]:c.rowptr[i + 1]], c.counts[c.rowptr[i]:c.rowptr[i + 1]]
        b = c.ids[c.rowptr[j]:c.rowptr[j + 1]], c.counts[c.rowptr[j]:c.rowptr[j + 1]]
        a = [np.ascontiguousarray(v) for v in a]
        b = [np.ascontiguousarray(v) for v in b]
        want = R.ref_cosine(a[0].ctypes.data_as(U32), a[1].ctypes.data_as(U32), len(a[0]), b[0].ctypes.data_as(U32),
                            b[1].ctypes.data_as(U32), len(b[0]))
        assert got[q] == want


def test_simhash_equals_reference_md5_words():
    from tests.golden.make_golden import ref_hash, ref_simhash_words, term_word
    rng = np.random.default_rng(5)
    V = 300
    table = np.array([ref_hash(R, term_word(t)) for t in range(V)], np.uint64)
    lens = rng.integers(0, 80, 50)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    tok = rng.integers(0, V, int(off[-1]), dtype=np.uint32)
    c = oracle.count(tok, off, threads=1)
    fp = oracle.simhash(c, None, table=table, threads=2)
    for d in range(len(lens)):
        words = [term_word(int(t)) for t in tok[off[d]:off[d + 1]]]
        assert int(fp[d]) == ref_simhash_words(R, words)


def test_hamming_equals_reference():
    rng = np.random.default_rng(9)
    fp = rng.integers(0, 2**63, 200, dtype=np.uint64)
    fp[5] = fp[6] ^ np.uint64(0b1011)
    pairs = oracle.hamming_pairs(fp, 3, threads=2)
    got = {int(k) for k in pairs}
    want = {(i << 32) | j for i in range(200) for j in range(i + 1, 200) if R.ref_hamming(int(fp[i]), int(fp[j])) <= 3}
    assert got == want
