"""f4 on-disk formats: frequency table TSV,
MRCREF reference file, MRCS signature file, the
reference builders — host logic, CPU only. The SPEC's own
examples are the known answers; cf/df for the text examples come from the
oracle's extract_3grams restatement, itself pinned against the reference
(tests/test_text_oracle.py)."""
import struct

import numpy as np
import pytest

import oracle
from paper_1810_03099_b200 import ValidationError
from paper_1810_03099_b200 import formats as F


def cf_df_of_texts(docs):
    text = np.frombuffer(b"".join(d.encode() for d in docs), np.uint8) if any(docs) else np.zeros(0, np.uint8)
    off = np.zeros(len(docs) + 1, np.uint64)
    off[1:] = np.cumsum([len(d) for d in docs])
    tok, goff = oracle.text_grams(text, off)
    cf = np.bincount(tok, minlength=F.GRAM_SPACE).astype(np.uint64)
    df = np.zeros(F.GRAM_SPACE, np.uint64)
    for d in range(len(docs)):
        df[np.unique(tok[int(goff[d]):int(goff[d + 1])])] += 1
    return cf, df


# -- grams / hashing ------------------------------------------------------------
def test_gram_packing_is_lexicographic():
    assert F.pack_gram("aaa") == 0 and F.pack_gram("zzz") == F.GRAM_SPACE - 1
    assert F.pack_gram("the") == (19 * 26 + 7) * 26 + 4
    ids = np.arange(F.GRAM_SPACE)
    strs = [F.unpack_gram(i) for i in ids]
    assert strs == sorted(strs) and all(F.pack_gram(s) == i for i, s in zip(ids, strs))
    for bad in ["ab", "abcd", "aBc", "ab1", ""]:
        with pytest.raises(ValidationError):
            F.pack_gram(bad)


def test_fnv1a64_known_answers():
    assert F.fnv1a64(b"") == 0xCBF29CE484222325
    assert F.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert F.fnv1a64(b"foobar") == 0x85944171F73967E8


# -- frequency table -----------------------------------------------------------
def test_frequency_table_spec_examples():
    t = F.FrequencyTable.from_counts(*cf_df_of_texts(["abcd", "abcx"]))
    assert t.rows() == [("abc", 2, 2), ("bcd", 1, 1), ("bcx", 1, 1)]
    t = F.FrequencyTable.from_counts(*cf_df_of_texts(["aaaa"]))
    assert t.rows() == [("aaa", 2, 1)]
    t = F.FrequencyTable.from_counts(*cf_df_of_texts(["ab cd", "x y"]))
    assert len(t) == 0


def test_frequency_table_invariants_on_text():
    rng = np.random.default_rng(3)
    words = ["the", "and", "tion", "qzx", "ab", "jjq", "zzzz", "mrc"]
    docs = [" ".join(rng.choice(words, rng.integers(0, 30))) for _ in range(40)]
    cf, df = cf_df_of_texts(docs)
    t = F.FrequencyTable.from_counts(cf, df)
    tok, _ = oracle.text_grams(np.frombuffer("".join(docs).encode(), np.uint8),
                               np.r_[0, np.cumsum([len(d) for d in docs])].astype(np.uint64))
    assert int(t.cf.sum()) == len(tok)
    assert np.all(t.df >= 1) and np.all(t.df <= len(docs)) and np.all(t.cf >= t.df)
    key = [(-int(c), int(g)) for g, c in zip(t.gram, t.cf)]
    assert key == sorted(key)


def test_frequency_table_round_trip(tmp_path):
    t = F.FrequencyTable.from_rows([("abc", 2, 2), ("bcd", 1, 1), ("bcx", 1, 1)])
    F.save_frequency_table(t, tmp_path / "t.tsv")
    assert (tmp_path / "t.tsv").read_text() == "abc\t2\t2\nbcd\t1\t1\nbcx\t1\t1\n"
    assert F.load_frequency_table(tmp_path / "t.tsv") == t
    rng = np.random.default_rng(11)
    for case in range(100):  # 100 randomized cases
        n = int(rng.integers(0, 300))
        g = rng.choice(F.GRAM_SPACE, n, replace=False)
        df = rng.integers(1, 1000, n).astype(np.uint64)
        cf = df + rng.integers(0, 1 << 40, n).astype(np.uint64) * (case % 2)
        dense_cf = np.zeros(F.GRAM_SPACE, np.uint64)
        dense_df = np.zeros(F.GRAM_SPACE, np.uint64)
        dense_cf[g], dense_df[g] = cf, df
        t = F.FrequencyTable.from_counts(dense_cf, dense_df)
        assert F.loads_frequency_table(F.dumps_frequency_table(t)) == t


def test_frequency_table_comments_and_errors():
    t = F.loads_frequency_table("# gram\tcf\tdf\nabc\t2\t2\n#x\nbcd\t1\t1\n")
    assert t.rows() == [("abc", 2, 2), ("bcd", 1, 1)]
    cases = {
        "abc\t2\t2\nab\t5\t2\n": "gram length ≠ 3 at line 2",
        "abc\t2\n": "wrong field count (2, expected 3) at line 1",
        "abc\t2\t2\t1\n": "wrong field count (4, expected 3) at line 1",
        "abc\tx\t2\n": "non-integer frequency at line 1",
        "abc\t2\t-1\n": "non-integer frequency at line 1",
        "aBc\t2\t2\n": "is not 3 lowercase letters at line 1",
        "abc\t1\t2\n": "need corpus_freq >= doc_freq >= 1 at line 1",
        "abc\t3\t0\n": "need corpus_freq >= doc_freq >= 1 at line 1",
        "abc\t2\t2\nabc\t1\t1\n": "duplicate gram at line 2",
        "abc\t1\t1\nbcd\t2\t1\n": "rows not sorted",
        "bcd\t1\t1\nabc\t1\t1\n": "rows not sorted",
    }
    for text, msg in cases.items():
        with pytest.raises(ValidationError, match=msg.replace("(", r"\(").replace(")", r"\)")):
            F.loads_frequency_table(text)


# -- reference builders and partitions -----------------------------------------
def small_table():
    return F.FrequencyTable.from_rows([("abc", 5, 3), ("qzx", 1, 1), ("jjq", 2, 1), ("the", 100, 9),
                                       ("and", 90, 8)])


def test_builders_spec_examples():
    a = F.build_all()
    assert len(a) == 17576 and F.unpack_gram(a.grams[0]) == "aaa" and F.unpack_gram(a.grams[-1]) == "zzz"
    assert int(np.sum(a.grams == F.pack_gram("the"))) == 1
    t = small_table()
    nz = F.build_nonzero(t)
    assert [F.unpack_gram(g) for g in nz.grams] == ["the", "and", "abc", "jjq", "qzx"]
    assert F.build_band(t, 0, len(t)).grams.tolist() == nz.grams.tolist()
    assert [F.unpack_gram(g) for g in F.build_band(t, 0, 2).grams] == ["the", "and"]
    with pytest.raises(ValidationError, match="exceeds the nonzero list length 5"):
        F.build_band(t, 0, 9999)
    ig = F.build_infogain(F.FrequencyTable.from_rows([("abc", 5, 3), ("qzx", 1, 1), ("jjq", 2, 1)]), 2)
    assert [F.unpack_gram(g) for g in ig.grams] == ["qzx", "jjq"]
    ig = F.build_infogain(t, 4)  # df==1 exhausted -> extend with higher df, same ordering
    assert [F.unpack_gram(g) for g in ig.grams] == ["qzx", "jjq", "abc", "and"]
    with pytest.raises(ValidationError, match="exceeds the 5 grams"):
        F.build_infogain(t, 6)


def test_infogain_prefers_unique_grams_brute_force():
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = 200
        g = rng.choice(F.GRAM_SPACE, n, replace=False)
        df = rng.integers(1, 4, n)
        cf = df + rng.integers(0, 5, n)
        t = F.FrequencyTable.from_rows([(F.unpack_gram(a), int(b), int(c)) for a, b, c in zip(g, cf, df)])
        k = int(rng.integers(1, n))
        out = set(F.build_infogain(t, k).grams.tolist())
        ranked = sorted(zip(df, cf, [F.unpack_gram(x) for x in g]))
        assert out == {F.pack_gram(s) for _, _, s in ranked[:k]}
        if k <= int(np.sum(df == 1)):
            assert all(d == 1 for d, gg in zip(df, g) if int(gg) in out)


def test_partition_ceil_rule():
    gl = F.GramList(np.arange(10, dtype=np.uint32), "all")
    assert F.partition(gl, 3).sizes == [4, 4, 2]
    assert F.partition(gl, 1).sizes == [10]
    assert F.partition(F.GramList(np.arange(1500, dtype=np.uint32), "infogain(1500)"), 60).sizes == [25] * 60
    r = F.partition(gl, 3)
    parts = r.partitions
    assert np.array_equal(np.concatenate(parts), gl.grams) and [len(p) for p in parts] == [4, 4, 2]
    assert r.rowptr.tolist() == [0, 4, 8, 10]
    for p in (0, 11):
        with pytest.raises(ValidationError, match="outside"):
            F.partition(gl, p)
    with pytest.raises(ValidationError, match="last partition empty"):
        F.partition(F.GramList(np.arange(9, dtype=np.uint32), "all"), 4)
    with pytest.raises(ValidationError, match="distinct"):
        F.partition(F.GramList(np.array([1, 2, 1], np.uint32), "all"), 1)


# -- MRCREF ---------------------------------------------------------------------------
def test_mrcref_format_and_round_trip(tmp_path):
    r = F.partition(F.GramList(np.array([F.pack_gram(s) for s in ["the", "and", "qzx"]], np.uint32), "nonzero"), 2)
    assert F.dumps_reference(r) == "MRCREF 1 2 3 nonzero\nthe\nand\nqzx\n"
    F.save_reference(r, tmp_path / "r.ref")
    r2 = F.load_reference(tmp_path / "r.ref")
    assert r2 == r and r2.sizes == [2, 1] and r2.ref_id == r.ref_id == F.fnv1a64((tmp_path / "r.ref").read_bytes())
    rng = np.random.default_rng(7)
    for _ in range(100):
        L = int(rng.integers(1, 2000))
        g = rng.choice(F.GRAM_SPACE, L, replace=False).astype(np.uint32)
        c = int(rng.integers(1, L + 1))
        P = next(p for p in range(c, 0, -1) if -(-L // p) * (p - 1) < L)
        prov = rng.choice(["all", "nonzero", f"band(0,{L})", f"infogain({L})"])
        r = F.partition(F.GramList(g, str(prov)), P)
        r2 = F.loads_reference(F.dumps_reference(r))
        assert r2 == r and r2.sizes == r.sizes and r2.ref_id == r.ref_id


def test_mrcref_errors():
    cases = {
        "MRCREF 1 2 2 all\nabc\nabc\n": "duplicate gram at line 3",
        "MRCREF 1 0 2 all\nabc\nabd\n": "P=0 must be >= 1",
        "MRCX 1 1 1 all\nabc\n": "bad magic",
        "MRCREF 2 1 1 all\nabc\n": "unsupported MRCREF version",
        "MRCREF 1 1 3 all\nabc\nabd\n": "gram-count mismatch: header L=3, file has 2",
        "MRCREF 1 1 1 all\nab\n": 'not a 3-gram "ab" at line 2',
        "MRCREF 1 3 2 all\nabc\nabd\n": "outside",
        "MRCREF 1 1 1\nabc\n": "header needs 5 fields",
        "": "empty reference file",
    }
    for text, msg in cases.items():
        with pytest.raises(ValidationError, match=msg.replace("(", r"\(")):
            F.loads_reference(text)


# -- MRCS -----------------------------------------------------------------------------
def test_mrcs_layout_and_round_trip(tmp_path):
    v = np.array([0.5, 0.0, 1.0 / 3.0])
    b = F.encode_signature(v, 0x0123456789ABCDEF)
    assert b[:4] == b"MRCS" and struct.unpack_from("<IIQ", b, 4) == (1, 3, 0x0123456789ABCDEF)
    assert len(b) == 20 + 8 * 3 and np.frombuffer(b, "<f8", 3, 20).tolist() == v.tolist()
    assert len(F.encode_signature(np.zeros(30), 1)) - 20 == 240  # SPEC §6 byte counts, P=30/60
    assert len(F.encode_signature(np.zeros(60), 1)) - 20 == 480
    F.save_signature(tmp_path / "d.mrcs", v, 42)
    v2, rid = F.load_signature(tmp_path / "d.mrcs")
    assert rid == 42 and v2.tobytes() == v.tobytes()
    rng = np.random.default_rng(9)
    for _ in range(100):
        P = int(rng.integers(1, 300))
        v = rng.random(P)
        v[rng.random(P) < 0.2] = 0.0
        rid = int(rng.integers(0, 1 << 63)) * 2 + 1
        v2, rid2 = F.decode_signature(F.encode_signature(v, rid))
        assert rid2 == rid and v2.tobytes() == v.tobytes()


def test_mrcs_errors_and_records():
    b = F.encode_signature(np.ones(4), 5)
    with pytest.raises(ValidationError, match="bad magic"):
        F.decode_signature(b"XRCS" + b[4:])
    with pytest.raises(ValidationError, match="unsupported MRCS version 2"):
        F.decode_signature(b[:4] + struct.pack("<I", 2) + b[8:])
    with pytest.raises(ValidationError, match="MRCS size"):
        F.decode_signature(b[:-8])
    with pytest.raises(ValidationError, match="ref_id mismatch"):
        F.check_same_reference(1, 2)
    F.check_same_reference(7, 7)
    S = np.random.default_rng(1).random((5, 4))
    rec = np.stack([np.frombuffer(F.encode_signature(S[i], 100 + i), np.uint8) for i in range(5)])
    S2, ids = F.decode_records(rec)
    assert S2.tobytes() == S.tobytes() and ids.tolist() == [100, 101, 102, 103, 104]
    bad = rec.copy()
    bad[2, 0] = ord("X")
    with pytest.raises(ValidationError, match="malformed MRCS record"):
        F.decode_records(bad)
