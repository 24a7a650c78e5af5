"""CPU oracle for the MRC batch-similarity path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or the
timed CPU baseline. The product (paper_1810_03099_b200) never imports it.

liboracle.so is the C++ restatement (oracle/oracle.cpp, each function citing
the reference file:line it follows). librefshim.so (oracle/_ref/, built by
`make ref` from the reference's own headers under /root/reference) exposes the
reference's NgramVector::from_entries, cosine, word_hash64, simhash and
hamming so the restatement can be pinned against the real code.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
P = ctypes.POINTER
u8p = P(ctypes.c_uint8)
u32p = P(ctypes.c_uint32)
u64p = P(ctypes.c_uint64)
f32p = P(ctypes.c_float)
f64p = P(ctypes.c_double)


def _p(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(P(ct))


class _Pairs(ctypes.Structure):
    _fields_ = [("pairs", u64p), ("n_pairs", ctypes.c_uint64), ("border", u64p), ("n_border", ctypes.c_uint64)]


_orc = None
_ref = None


def lib():
    global _orc
    if _orc is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run make")
        L = ctypes.CDLL(path)
        L.orc_count.argtypes = [u32p, u64p, ctypes.c_uint32, u64p, u32p, u32p, ctypes.c_int]
        L.orc_count.restype = ctypes.c_uint64
        L.orc_df.argtypes = [u64p, u32p, ctypes.c_uint32, ctypes.c_uint32, u32p]
        L.orc_idf32.argtypes = [u32p, ctypes.c_uint32, ctypes.c_uint32, f32p]
        L.orc_weights.argtypes = [u64p, u32p, u32p, ctypes.c_uint32, f32p, f64p, f64p]
        L.orc_cosine.argtypes = [u32p, f64p, ctypes.c_uint64, ctypes.c_double, u32p, f64p, ctypes.c_uint64,
                                 ctypes.c_double]
        L.orc_cosine.restype = ctypes.c_double
        L.orc_sign.argtypes = [u64p, u32p, f64p, f64p, ctypes.c_uint32, u64p, u32p, f64p, f64p, ctypes.c_uint32,
                               f64p, ctypes.c_int]
        L.orc_compare.argtypes = [f64p, f64p, ctypes.c_uint32]
        L.orc_compare.restype = ctypes.c_double
        L.orc_pairs_free.argtypes = [P(_Pairs)]
        L.orc_mrc_pairs.argtypes = [f64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_uint32, ctypes.c_uint32, P(_Pairs), ctypes.c_int]
        L.orc_mrc_query_pairs.argtypes = [f64p, ctypes.c_uint32, f64p, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_double, ctypes.c_double, P(_Pairs), ctypes.c_int]
        L.orc_term_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        L.orc_term_hash.restype = ctypes.c_uint64
        L.orc_simhash.argtypes = [u64p, u32p, u32p, ctypes.c_uint32, f32p, ctypes.c_uint64, u64p, u64p, ctypes.c_int]
        L.orc_hamming_pairs.argtypes = [u64p, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                        P(_Pairs), ctypes.c_int]
        L.orc_hamming_query_pairs.argtypes = [u64p, ctypes.c_uint32, u64p, ctypes.c_uint32, ctypes.c_int, P(_Pairs),
                                              ctypes.c_int]
        L.orc_exact_pairs.argtypes = [u64p, u32p, f64p, f64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_uint32, ctypes.c_uint32, P(_Pairs), ctypes.c_int]
        L.orc_cosine_pairs.argtypes = [u64p, u32p, f64p, f64p, u64p, ctypes.c_uint64, f64p, ctypes.c_int]
        u8p = P(ctypes.c_uint8)
        L.orc_text_grams.argtypes = [u8p, u64p, ctypes.c_uint32, u32p, u64p]
        L.orc_text_grams.restype = ctypes.c_uint64
        L.orc_word_hash64.argtypes = [u8p, ctypes.c_uint64]
        L.orc_word_hash64.restype = ctypes.c_uint64
        L.orc_text_simhash.argtypes = [u8p, u64p, ctypes.c_uint32, u64p, ctypes.c_int]
        L.orc_evaluate.argtypes = [u64p, u32p, f64p, f64p, ctypes.c_uint32, f64p, ctypes.c_uint32, u64p,
                                   ctypes.c_uint32, ctypes.c_uint32, f64p, ctypes.c_int]
        _orc = L
    return _orc


def ref_lib():
    """The reference's own code (oracle/_ref/librefshim.so) or None if not built."""
    global _ref
    if _ref is None:
        path = os.path.join(_HERE, "_ref", "librefshim.so")
        if not os.path.exists(path):
            return None
        L = ctypes.CDLL(path)
        L.ref_from_entries.argtypes = [u32p, u32p, ctypes.c_uint64, u32p, u32p, f64p]
        L.ref_from_entries.restype = ctypes.c_uint64
        L.ref_cosine.argtypes = [u32p, u32p, ctypes.c_uint64, u32p, u32p, ctypes.c_uint64]
        L.ref_cosine.restype = ctypes.c_double
        L.ref_extract_3grams.argtypes = [ctypes.c_char_p, ctypes.c_uint64, u32p, u32p, ctypes.c_uint64]
        L.ref_extract_3grams.restype = ctypes.c_uint64
        L.ref_normalize.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_normalize.restype = ctypes.c_uint64
        L.ref_word_hash64.argtypes = [ctypes.c_char_p, ctypes.c_uint64, P(ctypes.c_int)]
        L.ref_word_hash64.restype = ctypes.c_uint64
        L.ref_simhash.argtypes = [ctypes.c_char_p, u64p, ctypes.c_uint64]
        L.ref_simhash.restype = ctypes.c_uint64
        L.ref_hamming.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ref_hamming.restype = ctypes.c_int
        L.ref_pack_gram.argtypes = [ctypes.c_char_p, ctypes.c_uint64]
        L.ref_pack_gram.restype = ctypes.c_int64
        _ref = L
    return _ref


def _take_pairs(pr: _Pairs):
    n, b = pr.n_pairs, pr.n_border
    pairs = np.ctypeslib.as_array(pr.pairs, shape=(max(n, 1),))[:n].copy() if n else np.zeros(0, np.uint64)
    border = np.ctypeslib.as_array(pr.border, shape=(max(b, 1),))[:b].copy() if b else np.zeros(0, np.uint64)
    lib().orc_pairs_free(ctypes.byref(pr))
    return pairs, border


@dataclass
class Counts:
    rowptr: np.ndarray
    ids: np.ndarray
    counts: np.ndarray

    @property
    def n_docs(self):
        return len(self.rowptr) - 1


def count(tokens: np.ndarray, doc_off: np.ndarray, threads: int = 0) -> Counts:
    n = len(doc_off) - 1
    T = int(doc_off[-1])
    rowptr = np.zeros(n + 1, np.uint64)
    ids = np.empty(max(T, 1), np.uint32)
    cnt = np.empty(max(T, 1), np.uint32)
    tokens = np.ascontiguousarray(tokens, np.uint32)
    doc_off = np.ascontiguousarray(doc_off, np.uint64)
    nnz = lib().orc_count(_p(tokens, ctypes.c_uint32), _p(doc_off, ctypes.c_uint64), n, _p(rowptr, ctypes.c_uint64),
                          _p(ids, ctypes.c_uint32), _p(cnt, ctypes.c_uint32), threads)
    return Counts(rowptr, ids[:nnz].copy(), cnt[:nnz].copy())


def df(c: Counts, vocab: int) -> np.ndarray:
    out = np.empty(vocab, np.uint32)
    lib().orc_df(_p(c.rowptr, ctypes.c_uint64), _p(c.ids, ctypes.c_uint32), c.n_docs, vocab, _p(out, ctypes.c_uint32))
    return out


def idf32(dfv: np.ndarray, n_docs: int) -> np.ndarray:
    out = np.empty(len(dfv), np.float32)
    lib().orc_idf32(_p(dfv, ctypes.c_uint32), n_docs, len(dfv), _p(out, ctypes.c_float))
    return out


def weights(c: Counts, idf: np.ndarray | None):
    w = np.empty(max(len(c.ids), 1), np.float64)
    nrm = np.empty(c.n_docs, np.float64)
    lib().orc_weights(_p(c.rowptr, ctypes.c_uint64), _p(c.ids, ctypes.c_uint32), _p(c.counts, ctypes.c_uint32),
                      c.n_docs, _p(idf, ctypes.c_float) if idf is not None else None, _p(w, ctypes.c_double),
                      _p(nrm, ctypes.c_double))
    return w[: len(c.ids)], nrm


@dataclass
class Weighted:
    rowptr: np.ndarray
    ids: np.ndarray
    w: np.ndarray
    norm: np.ndarray

    @property
    def n_docs(self):
        return len(self.rowptr) - 1


def weighted(c: Counts, idf: np.ndarray | None) -> Weighted:
    w, nrm = weights(c, idf)
    return Weighted(c.rowptr, c.ids, w, nrm)


def rows(x: Weighted, docs) -> Weighted:
    """Sub-CSR of the given docs (e.g. the K reference docs)."""
    rp = [0]
    ids, w = [], []
    for d in docs:
        b, e = int(x.rowptr[d]), int(x.rowptr[d + 1])
        ids.append(x.ids[b:e])
        w.append(x.w[b:e])
        rp.append(rp[-1] + e - b)
    return Weighted(np.array(rp, np.uint64), np.concatenate(ids).astype(np.uint32) if ids else np.zeros(0, np.uint32),
                    np.concatenate(w) if w else np.zeros(0), x.norm[np.asarray(docs, dtype=np.int64)].copy())


def vectors(rowptr, ids, w) -> Weighted:
    """Explicit reference vectors (e.g. partitions with weight 1)."""
    rowptr = np.asarray(rowptr, np.uint64)
    ids = np.asarray(ids, np.uint32)
    w = np.asarray(w, np.float64)
    nrm = np.array([np.sqrt(np.sum(w[int(rowptr[k]):int(rowptr[k + 1])] ** 2)) for k in range(len(rowptr) - 1)])
    # the merge-join needs ids sorted within each vector
    ids2, w2 = ids.copy(), w.copy()
    for k in range(len(rowptr) - 1):
        b, e = int(rowptr[k]), int(rowptr[k + 1])
        o = np.argsort(ids[b:e], kind="stable")
        ids2[b:e] = ids[b:e][o]
        w2[b:e] = w[b:e][o]
    return Weighted(rowptr, ids2, w2, nrm)


def sign(x: Weighted, ref: Weighted, threads: int = 0) -> np.ndarray:
    K = ref.n_docs
    S = np.empty((x.n_docs, K), np.float64)
    lib().orc_sign(_p(x.rowptr, ctypes.c_uint64), _p(x.ids, ctypes.c_uint32), _p(x.w, ctypes.c_double),
                   _p(x.norm, ctypes.c_double), x.n_docs, _p(ref.rowptr, ctypes.c_uint64),
                   _p(ref.ids, ctypes.c_uint32), _p(ref.w, ctypes.c_double), _p(ref.norm, ctypes.c_double), K,
                   _p(S, ctypes.c_double), threads)
    return S


def compare(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().orc_compare(_p(a, ctypes.c_double), _p(b, ctypes.c_double), len(a))


def mrc_pairs(S: np.ndarray, tau: float, band: float = 1e-5, row_lo: int = 0, row_hi: int | None = None,
              threads: int = 0):
    S = np.ascontiguousarray(S, np.float64)
    n, K = S.shape
    pr = _Pairs()
    lib().orc_mrc_pairs(_p(S, ctypes.c_double), n, K, tau, band, row_lo, n if row_hi is None else row_hi,
                        ctypes.byref(pr), threads)
    return _take_pairs(pr)


def evaluate(x: Weighted, S: np.ndarray, fp: np.ndarray | None = None, row_lo: int = 0,
             row_hi: int | None = None, threads: int = 0) -> dict:
    """SPEC eval (Eq. 2/3) over pairs i<j of rows [row_lo, row_hi): MAE, mean
    error and variance of MRC (and Simhash) against the exact cosine."""
    S = np.ascontiguousarray(S, np.float64)
    n, K = S.shape
    out = np.zeros(7, np.float64)
    fpa = None if fp is None else np.ascontiguousarray(fp, np.uint64)
    lib().orc_evaluate(_p(x.rowptr, ctypes.c_uint64), _p(x.ids, ctypes.c_uint32), _p(x.w, ctypes.c_double),
                       _p(x.norm, ctypes.c_double), n, _p(S, ctypes.c_double), K, _p(fpa, ctypes.c_uint64), row_lo,
                       n if row_hi is None else row_hi, _p(out, ctypes.c_double), threads)
    m = out[0]
    res = {"pairs": int(m)}
    for name, o in (("mrc", 1), ("simhash", 4)):
        mean = out[o] / m
        res[name + "_mae"] = out[o + 2] / m
        res[name + "_mean_error"] = mean
        res[name + "_variance"] = max(0.0, out[o + 1] / m - mean * mean)
    if fp is None:
        for k in ("simhash_mae", "simhash_mean_error", "simhash_variance"):
            res[k] = float("nan")
    return res


def mrc_query_pairs(Sq, Sd, tau: float, band: float = 1e-5, threads: int = 0):
    Sq = np.ascontiguousarray(Sq, np.float64)
    Sd = np.ascontiguousarray(Sd, np.float64)
    pr = _Pairs()
    lib().orc_mrc_query_pairs(_p(Sq, ctypes.c_double), Sq.shape[0], _p(Sd, ctypes.c_double), Sd.shape[0],
                              Sq.shape[1], tau, band, ctypes.byref(pr), threads)
    return _take_pairs(pr)


def term_hash(seed: int, t: int) -> int:
    return lib().orc_term_hash(seed, t)


def simhash(c: Counts, idf: np.ndarray | None, seed: int = 0, table: np.ndarray | None = None,
            threads: int = 0) -> np.ndarray:
    fp = np.empty(c.n_docs, np.uint64)
    lib().orc_simhash(_p(c.rowptr, ctypes.c_uint64), _p(c.ids, ctypes.c_uint32), _p(c.counts, ctypes.c_uint32),
                      c.n_docs, _p(idf, ctypes.c_float) if idf is not None else None, seed,
                      _p(table, ctypes.c_uint64) if table is not None else None, _p(fp, ctypes.c_uint64), threads)
    return fp


def text_grams(text: np.ndarray, off: np.ndarray):
    """3-gram id stream per doc of raw text bytes (ngram.hpp:114-180):
    (tokens u32, gram_off u64[n+1]); vocabulary 26^3 = 17576."""
    text = np.ascontiguousarray(text, np.uint8)
    off = np.ascontiguousarray(off, np.uint64)
    n = len(off) - 1
    gram_off = np.empty(n + 1, np.uint64)
    tot = lib().orc_text_grams(_p(text, ctypes.c_uint8), _p(off, ctypes.c_uint64), n, None,
                               _p(gram_off, ctypes.c_uint64))
    tokens = np.empty(max(tot, 1), np.uint32)
    lib().orc_text_grams(_p(text, ctypes.c_uint8), _p(off, ctypes.c_uint64), n, _p(tokens, ctypes.c_uint32),
                         _p(gram_off, ctypes.c_uint64))
    return tokens[:tot], gram_off


def word_hash64(word: bytes) -> int:
    """First 8 bytes of MD5(word), big-endian (simhash.hpp:23-29)."""
    b = np.frombuffer(word, np.uint8) if len(word) else np.zeros(1, np.uint8)
    return int(lib().orc_word_hash64(_p(np.ascontiguousarray(b), ctypes.c_uint8), len(word)))


def text_simhash(text: np.ndarray, off: np.ndarray, threads: int = 0) -> np.ndarray:
    """simhash(extract_words(normalize(doc))) per doc (simhash.hpp:35-45)."""
    text = np.ascontiguousarray(text, np.uint8)
    off = np.ascontiguousarray(off, np.uint64)
    fp = np.empty(len(off) - 1, np.uint64)
    lib().orc_text_simhash(_p(text, ctypes.c_uint8), _p(off, ctypes.c_uint64), len(off) - 1, _p(fp, ctypes.c_uint64),
                           threads)
    return fp


def hamming_pairs(fp: np.ndarray, max_dist: int, row_lo: int = 0, row_hi: int | None = None, threads: int = 0):
    fp = np.ascontiguousarray(fp, np.uint64)
    pr = _Pairs()
    n = len(fp)
    lib().orc_hamming_pairs(_p(fp, ctypes.c_uint64), n, max_dist, row_lo, n if row_hi is None else row_hi,
                            ctypes.byref(pr), threads)
    return _take_pairs(pr)[0]


def hamming_query_pairs(fq, fd, max_dist: int, threads: int = 0):
    fq = np.ascontiguousarray(fq, np.uint64)
    fd = np.ascontiguousarray(fd, np.uint64)
    pr = _Pairs()
    lib().orc_hamming_query_pairs(_p(fq, ctypes.c_uint64), len(fq), _p(fd, ctypes.c_uint64), len(fd), max_dist,
                                  ctypes.byref(pr), threads)
    return _take_pairs(pr)[0]


def exact_pairs(x: Weighted, vocab: int, tau: float, band: float = 1e-5, row_lo: int = 0,
                row_hi: int | None = None, threads: int = 0):
    pr = _Pairs()
    n = x.n_docs
    lib().orc_exact_pairs(_p(x.rowptr, ctypes.c_uint64), _p(x.ids, ctypes.c_uint32), _p(x.w, ctypes.c_double),
                          _p(x.norm, ctypes.c_double), n, vocab, tau, band, row_lo, n if row_hi is None else row_hi,
                          ctypes.byref(pr), threads)
    return _take_pairs(pr)


def cosine_pairs(x: Weighted, keys: np.ndarray, threads: int = 0) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint64)
    out = np.empty(len(keys), np.float64)
    lib().orc_cosine_pairs(_p(x.rowptr, ctypes.c_uint64), _p(x.ids, ctypes.c_uint32), _p(x.w, ctypes.c_double),
                           _p(x.norm, ctypes.c_double), _p(keys, ctypes.c_uint64), len(keys),
                           _p(out, ctypes.c_double), threads)
    return out


@dataclass
class MrcResult:
    counts: Counts
    df: np.ndarray
    idf: np.ndarray | None
    x: Weighted
    S: np.ndarray


def mrc_pipeline(tokens, doc_off, vocab: int, ref_docs, weighting: str = "tfidf", threads: int = 0) -> MrcResult:
    """count -> df -> idf -> weights -> sign in the oracle."""
    c = count(tokens, doc_off, threads)
    d = df(c, vocab)
    idf = idf32(d, c.n_docs) if weighting == "tfidf" else None
    x = weighted(c, idf)
    ref = rows(x, ref_docs)
    S = sign(x, ref, threads)
    return MrcResult(c, d, idf, x, S)
