"""Oracle vs the reference SPEC's known answers and the golden fixtures made
from the reference's own code (tests/golden/make_golden.py). CPU only."""
import math

import numpy as np
import pytest

import oracle


def gram(s):
    return (ord(s[0]) - 97) * 676 + (ord(s[1]) - 97) * 26 + (ord(s[2]) - 97)


def one_doc_counts(ids):
    toks = np.array(ids, np.uint32)
    return oracle.count(toks, np.array([0, len(toks)], np.uint64), threads=1)


def test_extract_counts_spec_examples(spec_examples):
    # SPEC.md:60-63 via the reference (golden): "abcabc" -> {abc:2,bca:1,cab:1}
    c = one_doc_counts([gram("abc"), gram("bca"), gram("cab"), gram("abc")])
    want = spec_examples["extract_3grams"]["abcabc"]
    assert [[int(i), int(n)] for i, n in zip(c.ids, c.counts)] == want
    c = one_doc_counts([gram("abc"), gram("bcd")])
    assert [[int(i), int(n)] for i, n in zip(c.ids, c.counts)] == spec_examples["extract_3grams"]["abcd"]


def test_cosine_spec_examples(spec_examples):
    # SPEC.md:78-81 (reference values: 0.49999999999999989, 1-2^-52.., 0)
    def wv(pairs):
        c = oracle.Counts(np.array([0, len(pairs)], np.uint64), np.array([p[0] for p in pairs], np.uint32),
                          np.array([p[1] for p in pairs], np.uint32))
        return oracle.weighted(c, None)

    a = wv([(gram("abc"), 1), (gram("bcd"), 1)])
    b = wv([(gram("bcd"), 1), (gram("cde"), 1)])
    ab2 = wv([(gram("abc"), 2), (gram("bca"), 1)])
    e = wv([])

    def cos(x, y):
        return oracle.lib().orc_cosine(oracle._p(x.ids, oracle.ctypes.c_uint32), oracle._p(x.w, oracle.ctypes.c_double),
                                       len(x.ids), float(x.norm[0]), oracle._p(y.ids, oracle.ctypes.c_uint32),
                                       oracle._p(y.w, oracle.ctypes.c_double), len(y.ids), float(y.norm[0]))

    # bit-identical to the reference's double arithmetic
    assert cos(a, b) == spec_examples["cosine"]["abc_bcd__bcd_cde"]
    assert cos(ab2, ab2) == spec_examples["cosine"]["identical"]
    assert cos(a, e) == 0.0 == spec_examples["cosine"]["with_empty"]
    assert abs(cos(a, b) - 0.5) <= 1e-12


def test_sign_spec_example(spec_examples):
    # partitions [{abc}],[{xyz}], doc "abcabc" -> [2/sqrt(6), 0]
    c = one_doc_counts([gram("abc"), gram("bca"), gram("cab"), gram("abc")])
    x = oracle.weighted(c, None)
    ref = oracle.vectors([0, 1, 2], [gram("abc"), gram("xyz")], [1.0, 1.0])
    S = oracle.sign(x, ref, threads=1)
    assert S[0, 0] == spec_examples["sign_abcabc"][0]
    assert S[0, 1] == 0.0
    assert abs(S[0, 0] - 2 / math.sqrt(6)) < 1e-12


def test_compare_spec_examples():
    # identical -> 1, orthogonal -> 0, all-zero -> 0
    s = np.array([0.3, 0.5, 0.1])
    assert abs(oracle.compare(s, s) - 1.0) < 1e-12
    e1 = np.zeros(5); e1[0] = 1
    e2 = np.zeros(5); e2[1] = 1
    assert oracle.compare(e1, e2) == 0.0
    assert oracle.compare(np.zeros(3), s) == 0.0


def test_hamming_and_simhash_spec_examples(spec_examples):
    # SPEC.md:143-146 through the oracle's pair sweep
    x = 0x0123456789ABCDEF
    fp = np.array([x, x, x ^ 0xFFFFFFFFFFFFFFFF, 0x0F, 0x00], np.uint64)
    pairs = oracle.hamming_pairs(fp, 4, threads=1)
    got = {(int(k) >> 32, int(k) & 0xFFFFFFFF) for k in pairs}
    assert (0, 1) in got and (3, 4) in got and (0, 2) not in got
    assert spec_examples["hamming"] == {"x_x": 0, "0f_00": 4, "x_notx": 64}
    # [w] -> word_hash64(w); [w,w] -> same; [] -> 0
    h = spec_examples["word_hash64"]["the"]
    table = np.zeros(4, np.uint64)
    table[2] = h
    c = oracle.Counts(np.array([0, 1, 2, 2], np.uint64), np.array([2, 2], np.uint32), np.array([1, 2], np.uint32))
    fps = oracle.simhash(c, None, table=table, threads=1)
    assert int(fps[0]) == h == spec_examples["simhash"]["single_the"]
    assert int(fps[1]) == h == spec_examples["simhash"]["double_the"]
    assert int(fps[2]) == 0 == spec_examples["simhash"]["empty"]


def test_oracle_counts_match_reference_golden(golden_small):
    g = golden_small
    c = oracle.count(g["tokens"], g["doc_off"], threads=2)
    assert np.array_equal(c.rowptr, g["rowptr"])
    assert np.array_equal(c.ids, g["ids"])
    assert np.array_equal(c.counts, g["counts"])
    _, nrm = oracle.weights(c, None)
    assert np.array_equal(nrm, g["norms"])  # ngram.hpp:100-104, bit-exact


def test_oracle_cosine_matches_reference_golden(golden_small):
    g = golden_small
    c = oracle.count(g["tokens"], g["doc_off"], threads=2)
    x = oracle.weighted(c, None)
    got = oracle.cosine_pairs(x, g["pair_keys"], threads=2)
    assert np.array_equal(got, g["pair_cos"])  # same merge-join order -> bit-exact


def test_oracle_sign_matches_reference_golden(golden_small):
    g = golden_small
    c = oracle.count(g["tokens"], g["doc_off"], threads=2)
    x = oracle.weighted(c, None)
    P = len(g["part_rowptr"]) - 1
    ref = oracle.vectors(g["part_rowptr"], g["part_ids"], np.ones(len(g["part_ids"])))
    S = oracle.sign(x, ref, threads=2)
    assert S.shape == (c.n_docs, P)
    np.testing.assert_allclose(S, g["sig_tf"], rtol=1e-12, atol=1e-15)


def test_oracle_simhash_matches_reference_golden(golden_small):
    g = golden_small
    c = oracle.count(g["tokens"], g["doc_off"], threads=2)
    fp = oracle.simhash(c, None, table=g["term_hash"], threads=2)
    assert np.array_equal(fp, g["fp_md5"])


def test_exact_inverted_index_equals_merge_join(golden_small):
    g = golden_small
    c = oracle.count(g["tokens"], g["doc_off"], threads=2)
    d = oracle.df(c, int(g["vocab"]))
    x = oracle.weighted(c, oracle.idf32(d, c.n_docs))
    pairs, border = oracle.exact_pairs(x, int(g["vocab"]), 0.05, threads=2)
    assert len(pairs) > 0
    cos = oracle.cosine_pairs(x, pairs, threads=2)
    assert np.all(cos >= 0.05)
    # every pair not listed is below tau (brute force over the triangle)
    n = c.n_docs
    iu = np.triu_indices(n, 1)
    allk = (iu[0].astype(np.uint64) << np.uint64(32)) | iu[1].astype(np.uint64)
    allc = oracle.cosine_pairs(x, allk, threads=2)
    assert np.array_equal(np.sort(allk[allc >= 0.05]), pairs)


def test_pair_count_arithmetic():
    # SPEC's 177,197,778 for 18,828 docs is wrong; C(n,2) is used.
    assert 18828 * 18827 // 2 == 177237378
    assert 18846 * 18845 // 2 == 177576435
