"""Synthetic corpora for BASELINE.json:configs[0..4] (input generation only).

The reference evaluates on NEWS20 (reference PAPER.md:219), which is absent;
seeded stand-ins with the configs' shapes replace it. The
generator is native (libmrcgen.so, include/mrcgen.h); this module binds it.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)
CONFIG_PATH = os.path.join(_REPO, "configs", "mrc_configs.json")


class _Spec(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("n_docs", ctypes.c_uint32),
        ("vocab", ctypes.c_uint32),
        ("n_topics", ctypes.c_uint32),
        ("len_min", ctypes.c_uint32),
        ("len_max", ctypes.c_uint32),
        ("_pad", ctypes.c_uint32),
        ("zipf_global", ctypes.c_double),
        ("zipf_topic", ctypes.c_double),
        ("topic_mix", ctypes.c_double),
        ("len_median", ctypes.c_double),
        ("len_sigma", ctypes.c_double),
        ("dup_rate", ctypes.c_double),
        ("resample_lo", ctypes.c_double),
        ("resample_hi", ctypes.c_double),
    ]


_lib = None


def _gen():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "lib", "libmrcgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (make)")
        lib = ctypes.CDLL(path)
        P = ctypes.POINTER
        lib.mrcgen_offsets.argtypes = [P(_Spec), P(ctypes.c_uint64)]
        lib.mrcgen_fill.argtypes = [P(_Spec), P(ctypes.c_uint64), P(ctypes.c_uint32), P(ctypes.c_uint32), ctypes.c_int]
        lib.mrcgen_offsets_queries.argtypes = [P(_Spec), P(_Spec), P(ctypes.c_uint64), P(ctypes.c_uint64)]
        lib.mrcgen_fill_queries.argtypes = [P(_Spec), P(_Spec), P(ctypes.c_uint64), P(ctypes.c_uint32),
                                            P(ctypes.c_uint64), P(ctypes.c_uint32), P(ctypes.c_uint32), ctypes.c_int]
        lib.mrcgen_sample_refs.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, P(ctypes.c_uint32)]
        lib.mrcgen_splitmix64_mix.argtypes = [ctypes.c_uint64]
        lib.mrcgen_splitmix64_mix.restype = ctypes.c_uint64
        lib.mrcgen_stream_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        lib.mrcgen_stream_seed.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def load_configs() -> dict:
    with open(CONFIG_PATH) as f:
        return json.load(f)


def spec_from_dict(d: dict) -> _Spec:
    s = _Spec()
    for k, v in d.items():
        setattr(s, k, v)
    return s


@dataclass
class Corpus:
    tokens: np.ndarray   # uint32 term ids, concatenated docs
    doc_off: np.ndarray  # uint64 [n_docs+1]
    vocab: int
    dup_src: np.ndarray  # uint32 [n_docs], 0xFFFFFFFF for originals

    @property
    def n_docs(self) -> int:
        return len(self.doc_off) - 1

    def slice_docs(self, n: int) -> "Corpus":
        """First n docs (a prefix keeps the generator's stream per doc)."""
        end = int(self.doc_off[n])
        return Corpus(self.tokens[:end].copy(), self.doc_off[: n + 1].copy(), self.vocab, self.dup_src[:n].copy())


def generate(spec: dict, threads: int = 0, pinned_tokens=None) -> Corpus:
    """Generate the corpus described by a configs/*.json 'corpus' dict."""
    lib = _gen()
    s = spec_from_dict(spec)
    n = s.n_docs
    off = np.zeros(n + 1, dtype=np.uint64)
    if lib.mrcgen_offsets(ctypes.byref(s), _ptr(off, ctypes.c_uint64)) != 0:
        raise ValueError("invalid corpus spec")
    T = int(off[-1])
    tokens = pinned_tokens if pinned_tokens is not None else np.empty(T, dtype=np.uint32)
    dup = np.empty(n, dtype=np.uint32)
    rc = lib.mrcgen_fill(ctypes.byref(s), _ptr(off, ctypes.c_uint64), _ptr(tokens, ctypes.c_uint32),
                         _ptr(dup, ctypes.c_uint32), threads)
    if rc != 0:
        raise ValueError("generator failed")
    return Corpus(tokens, off, s.vocab, dup)


def generate_queries(q_spec: dict, db_spec: dict, db: Corpus, threads: int = 0) -> Corpus:
    lib = _gen()
    q = spec_from_dict(q_spec)
    d = spec_from_dict(db_spec)
    off = np.zeros(q.n_docs + 1, dtype=np.uint64)
    if lib.mrcgen_offsets_queries(ctypes.byref(q), ctypes.byref(d), _ptr(db.doc_off, ctypes.c_uint64),
                                  _ptr(off, ctypes.c_uint64)) != 0:
        raise ValueError("invalid query spec")
    tokens = np.empty(int(off[-1]), dtype=np.uint32)
    src = np.empty(q.n_docs, dtype=np.uint32)
    rc = lib.mrcgen_fill_queries(ctypes.byref(q), ctypes.byref(d), _ptr(db.doc_off, ctypes.c_uint64),
                                 _ptr(db.tokens, ctypes.c_uint32), _ptr(off, ctypes.c_uint64),
                                 _ptr(tokens, ctypes.c_uint32), _ptr(src, ctypes.c_uint32), threads)
    if rc != 0:
        raise ValueError("query generator failed")
    return Corpus(tokens, off, q.vocab, src)


def sample_refs(seed: int, n: int, k: int) -> np.ndarray:
    """K distinct reference doc indices."""
    out = np.empty(k, dtype=np.uint32)
    if _gen().mrcgen_sample_refs(seed, n, k, _ptr(out, ctypes.c_uint32)) != 0:
        raise ValueError("bad reference sample arguments")
    return out


def config_corpus(name: str, threads: int = 0) -> tuple[Corpus, dict]:
    cfgs = load_configs()["configs"]
    c = cfgs[name]
    if "same_corpus_as" in c:
        base = cfgs[c["same_corpus_as"]]
        return generate(base["corpus"], threads), {**base, **c}
    return generate(c["corpus"], threads), c


# ---------------------------------------------------------------------------
# Synthetic raw text for the text front end (tests, bench). Each term id maps to
# a fixed pseudo-word (base-26 letters); words are joined by separators drawn
# from a seeded generator (spaces, punctuation, digits, newlines, a two-byte
# UTF-8 letter that the reference's ASCII normalize treats as a break), with
# some capitalised words. No dataset text is involved.
_SEPS = [b" ", b" ", b" ", b" ", b", ", b". ", b"\n", b" - ", b"; ", b" 42 ", b"\xc3\xa9", b"'", b"(", b") "]


def term_word(t: int) -> str:
    """Deterministic word for term id t: bijective base-26 letters (>= 1 char)."""
    s = ""
    t += 1
    while t > 0:
        t, r = divmod(t - 1, 26)
        s = chr(ord("a") + r) + s
    return s


def synth_text(tokens: np.ndarray, doc_off: np.ndarray, vocab: int, seed: int = 0):
    """(text uint8, byte_off uint64) with one word per token, vectorised."""
    rng = np.random.default_rng(seed)
    words = [term_word(t).encode() for t in range(vocab)]
    wlen = np.fromiter((len(w) for w in words), np.int64, vocab)
    wstart = np.zeros(vocab + 1, np.int64)
    np.cumsum(wlen, out=wstart[1:])
    wbytes = np.frombuffer(b"".join(words), np.uint8)
    sep_b = [np.frombuffer(x, np.uint8) for x in _SEPS]
    slen = np.array([len(x) for x in _SEPS], np.int64)
    sstart = np.zeros(len(_SEPS) + 1, np.int64)
    np.cumsum(slen, out=sstart[1:])
    sbytes = np.concatenate(sep_b)
    T = len(tokens)
    sep = rng.integers(0, len(_SEPS), T)
    tok = tokens.astype(np.int64)
    piece = wlen[tok] + slen[sep]
    pstart = np.zeros(T + 1, np.int64)
    np.cumsum(piece, out=pstart[1:])
    out = np.empty(pstart[-1], np.uint8)
    # word bytes
    wl = wlen[tok]
    idx = np.repeat(pstart[:-1], wl) + (np.arange(wl.sum()) - np.repeat(np.cumsum(wl) - wl, wl))
    src = np.repeat(wstart[tok], wl) + (np.arange(wl.sum()) - np.repeat(np.cumsum(wl) - wl, wl))
    out[idx] = wbytes[src]
    # separator bytes
    sl = slen[sep]
    idx = np.repeat(pstart[:-1] + wl, sl) + (np.arange(sl.sum()) - np.repeat(np.cumsum(sl) - sl, sl))
    src = np.repeat(sstart[sep], sl) + (np.arange(sl.sum()) - np.repeat(np.cumsum(sl) - sl, sl))
    out[idx] = sbytes[src]
    # capitalise ~10% of the words (first letter)
    cap = rng.random(T) < 0.1
    out[pstart[:-1][cap]] -= 32
    byte_off = pstart[doc_off.astype(np.int64)].astype(np.uint64)
    return out, byte_off
