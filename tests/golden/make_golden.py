"""Generate tests/golden/ fixtures from the REFERENCE's own code.

Runs in the dev container only (needs oracle/_ref/librefshim.so, built by
`make ref` from the reference headers under /root/reference). The outputs are
small committed fixtures; nothing on the GPU box reads /root/reference.

    python tests/golden/make_golden.py

Fixtures:
  spec_examples.json  reference outputs for the SPEC.md known answers on the
                      hot path (extract_3grams, cosine, word_hash64, simhash,
                      hamming, sign over partitions).
  corpus_small.npz    a seeded 300-doc corpus (configs[0] shape) with the
                      reference's per-doc NgramVector entries (from_entries),
                      raw-TF cosines (refsig::cosine) for sampled pairs,
                      TF signatures against 8 count-1 partition vectors
                      (SPEC.md:363 via refsig::cosine), and MD5-word Simhash
                      fingerprints (refsig::simhash over each doc's words).
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import oracle  # noqa: E402
from paper_1810_03099_b200 import corpus as C  # noqa: E402

U32 = ctypes.POINTER(ctypes.c_uint32)


def term_word(t: int) -> str:
    """Deterministic word for a synthetic term id: base-26 letters, >= 1 char."""
    s = ""
    t += 1
    while t > 0:
        t, r = divmod(t - 1, 26)
        s = chr(ord("a") + r) + s
    return s


def ref_counts(R, ids: np.ndarray):
    n = len(ids)
    oi = np.empty(max(n, 1), np.uint32)
    oc = np.empty(max(n, 1), np.uint32)
    nrm = ctypes.c_double()
    ids = np.ascontiguousarray(ids, np.uint32)
    k = R.ref_from_entries(ids.ctypes.data_as(U32), None, n, oi.ctypes.data_as(U32), oc.ctypes.data_as(U32),
                           ctypes.byref(nrm))
    return oi[:k].copy(), oc[:k].copy(), nrm.value


def ref_cos(R, ai, ac, bi, bc):
    return R.ref_cosine(ai.ctypes.data_as(U32), ac.ctypes.data_as(U32), len(ai), bi.ctypes.data_as(U32),
                        bc.ctypes.data_as(U32), len(bi))


def ref_extract(R, text: str):
    b = text.encode()
    cap = len(b) + 8
    oi = np.empty(cap, np.uint32)
    oc = np.empty(cap, np.uint32)
    k = R.ref_extract_3grams(b, len(b), oi.ctypes.data_as(U32), oc.ctypes.data_as(U32), cap)
    return [[int(i), int(c)] for i, c in zip(oi[:k], oc[:k])]


def ref_hash(R, w: str) -> int:
    err = ctypes.c_int()
    b = w.encode()
    return int(R.ref_word_hash64(b, len(b), ctypes.byref(err)))


def ref_simhash_words(R, words) -> int:
    packed = "".join(words).encode()
    lens = np.array([len(w.encode()) for w in words] or [0], np.uint64)
    return int(R.ref_simhash(packed, lens.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(words)))


def gram(s: str) -> int:
    return (ord(s[0]) - 97) * 676 + (ord(s[1]) - 97) * 26 + (ord(s[2]) - 97)


def main():
    R = oracle.ref_lib()
    if R is None:
        raise SystemExit("oracle/_ref/librefshim.so missing: run `make ref` first")

    # ---- SPEC known answers through the reference code -------------------
    spec = {}
    spec["extract_3grams"] = {t: ref_extract(R, t) for t in ["abcd", "ab cd", "abcabc", "Hello, World!", ""]}
    a = (np.array([gram("abc"), gram("bcd")], np.uint32), np.array([1, 1], np.uint32))
    b = (np.array([gram("bcd"), gram("cde")], np.uint32), np.array([1, 1], np.uint32))
    e = (np.array([], np.uint32), np.array([], np.uint32))
    ab2 = (np.array([gram("abc"), gram("bca")], np.uint32), np.array([2, 1], np.uint32))
    spec["cosine"] = {
        "abc_bcd__bcd_cde": ref_cos(R, *a, *b),
        "identical": ref_cos(R, *ab2, *ab2),
        "with_empty": ref_cos(R, *a, *e),
    }
    spec["word_hash64"] = {w: ref_hash(R, w) for w in ["a", "b", "the", "hello"]}
    spec["simhash"] = {
        "single_the": ref_simhash_words(R, ["the"]),
        "double_the": ref_simhash_words(R, ["the", "the"]),
        "empty": ref_simhash_words(R, []),
    }
    x = 0x0123456789ABCDEF
    spec["hamming"] = {"x_x": R.ref_hamming(x, x), "0f_00": R.ref_hamming(0x0F, 0), "x_notx": R.ref_hamming(
        x, x ^ 0xFFFFFFFFFFFFFFFF)}
    # sign example SPEC.md:366: partitions [{abc}],[{xyz}], doc "abcabc"
    doc = ref_counts(R, np.array([gram("abc"), gram("bca"), gram("cab"), gram("abc")], np.uint32))
    p1 = (np.array([gram("abc")], np.uint32), np.array([1], np.uint32))
    p2 = (np.array([gram("xyz")], np.uint32), np.array([1], np.uint32))
    spec["sign_abcabc"] = [ref_cos(R, doc[0], doc[1], *p1), ref_cos(R, doc[0], doc[1], *p2)]
    spec["grams"] = {"abc": gram("abc"), "bca": gram("bca"), "cab": gram("cab"), "xyz": gram("xyz")}
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(spec, f, indent=1, sort_keys=True)

    # ---- small seeded corpus ----------------------------------------------
    cfg = C.load_configs()["configs"]["c0"]["corpus"].copy()
    cfg["n_docs"] = 300
    cp = C.generate(cfg, threads=1)
    # add edge docs: an empty doc, a doc of one repeated term, a long (> 8192) doc
    rng = np.random.default_rng(7)
    extra = [np.zeros(0, np.uint32), np.full(17, 5, np.uint32),
             rng.integers(0, cfg["vocab"], 9000, dtype=np.uint32)]
    tokens = np.concatenate([cp.tokens] + extra)
    off = list(cp.doc_off.astype(np.uint64))
    for x_ in extra:
        off.append(off[-1] + len(x_))
    off = np.array(off, np.uint64)
    n = len(off) - 1
    V = cfg["vocab"]
    rows_ids, rows_cnt, norms = [], [], []
    rowptr = [0]
    for d in range(n):
        i, c, nr = ref_counts(R, tokens[off[d]:off[d + 1]])
        rows_ids.append(i)
        rows_cnt.append(c)
        norms.append(nr)
        rowptr.append(rowptr[-1] + len(i))
    ids = np.concatenate(rows_ids).astype(np.uint32)
    cnts = np.concatenate(rows_cnt).astype(np.uint32)
    # raw-TF cosines for sampled pairs (incl. the empty doc)
    pr = rng.integers(0, n, size=(2000, 2))
    pr = pr[pr[:, 0] != pr[:, 1]]
    pr.sort(axis=1)
    pr = np.unique(pr, axis=0)
    cos = np.array([ref_cos(R, rows_ids[i], rows_cnt[i], rows_ids[j], rows_cnt[j]) for i, j in pr])
    keys = (pr[:, 0].astype(np.uint64) << np.uint64(32)) | pr[:, 1].astype(np.uint64)
    # 8 count-1 partitions of the 400 most frequent terms (SPEC.md:306-314 ceil rule)
    freq = np.bincount(tokens, minlength=V)
    order = np.lexsort((np.arange(V), -freq))[:400]
    P = 8
    size = -(-len(order) // P)
    parts = [order[k * size:(k + 1) * size] for k in range(P)]
    part_rowptr = np.array([0] + list(np.cumsum([len(p) for p in parts])), np.uint64)
    part_ids = np.concatenate(parts).astype(np.uint32)
    sig = np.zeros((n, P))
    for d in range(n):
        for k, p in enumerate(parts):
            pi, pc, _ = ref_counts(R, p.astype(np.uint32))
            sig[d, k] = ref_cos(R, rows_ids[d], rows_cnt[d], pi, pc)
    # MD5-word simhash: words of term t repeated tf times, in any order
    table = np.array([ref_hash(R, term_word(t)) for t in range(V)], np.uint64)
    fps = np.array([ref_simhash_words(R, [term_word(int(t)) for t in tokens[off[d]:off[d + 1]]]) for d in range(n)],
                   np.uint64)
    np.savez_compressed(os.path.join(HERE, "corpus_small.npz"), tokens=tokens, doc_off=off, vocab=np.uint32(V),
                        rowptr=np.array(rowptr, np.uint64), ids=ids, counts=cnts, norms=np.array(norms),
                        pair_keys=keys, pair_cos=cos, part_rowptr=part_rowptr, part_ids=part_ids, sig_tf=sig,
                        term_hash=table, fp_md5=fps)
    print("wrote", os.listdir(HERE))


def text_fixture(R):
    """text_small.npz: seeded synthetic raw text (corpus.synth_text over a
    configs[0]-shaped corpus) plus edge documents, with the reference's
    extract_3grams(normalize(doc)) entries and simhash(words) per doc, and
    word_hash64 of words at the MD5 padding edges."""
    cfg = C.load_configs()["configs"]["c0"]["corpus"].copy()
    cfg["n_docs"] = 200
    cp = C.generate(cfg, threads=1)
    txt, off = C.synth_text(cp.tokens, cp.doc_off, cp.vocab, seed=7)
    docs = [bytes(txt[off[d]:off[d + 1]]) for d in range(cp.n_docs)]
    docs += [b"", b"!!! ... ,,, 123 456", b"AbC dEF-ghi", b"x" * 70 + b" " + b"y" * 55 + b"." + b"Z" * 56,
             "na\u00efve caf\u00e9 r\u00e9sum\u00e9 \u00fcber".encode(), b"ab", b"abc", b"a-b-c-d-e",
             b"The the THE tHe", b"  leading and trailing  ", b"q" * 64 + b"," + b"w" * 63 + b";" + b"e" * 65]
    text = np.frombuffer(b"".join(docs), np.uint8)
    boff = np.zeros(len(docs) + 1, np.uint64)
    np.cumsum([len(x) for x in docs], out=boff[1:])
    rowptr = [0]
    ids, cnts, fps = [], [], []
    for x in docs:
        cap = len(x) + 8
        oi = np.empty(cap, np.uint32)
        oc = np.empty(cap, np.uint32)
        k = R.ref_extract_3grams(x, len(x), oi.ctypes.data_as(U32), oc.ctypes.data_as(U32), cap)
        ids.append(oi[:k].copy())
        cnts.append(oc[:k].copy())
        rowptr.append(rowptr[-1] + k)
        nb = ctypes.create_string_buffer(len(x) + 1)
        m = R.ref_normalize(x, len(x), nb, len(x) + 1)
        words = [w for w in nb.raw[:m].decode().split(" ") if w]
        fps.append(ref_simhash_words(R, words))
    edge_words = ["a", "ab", "abc", "x" * 55, "x" * 56, "x" * 63, "x" * 64, "x" * 65, "y" * 119, "y" * 120,
                  "z" * 200]
    np.savez_compressed(os.path.join(HERE, "text_small.npz"), text=text, byte_off=boff,
                        rowptr=np.array(rowptr, np.uint64), ids=np.concatenate(ids).astype(np.uint32),
                        counts=np.concatenate(cnts).astype(np.uint32), fp=np.array(fps, np.uint64),
                        words=np.array(edge_words), word_hash=np.array([ref_hash(R, w) for w in edge_words],
                                                                       np.uint64))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "text":
        text_fixture(oracle.ref_lib())
    else:
        main()
        text_fixture(oracle.ref_lib())
