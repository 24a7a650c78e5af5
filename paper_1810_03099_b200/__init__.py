"""refsig-b200: B200-native MRC batch-similarity path (Python host binding).

Thin ctypes binding of the C ABI in include/refsig_gpu.h (librefsig_gpu.so,
CUDA kernels for sm_100a). It mirrors the reference's operations
(reference proj/include/refsig/*.hpp and SPEC.md signature/eval modules) as
batch calls over a whole corpus:

    count()              NgramVector::from_entries per doc (ngram.hpp:62-75)
    set_reference_*()    Reference.partition_vectors / K reference docs
    sign()               sign
    mrc_pairs(tau)       compare over all i<j
    simhash()            simhash (simhash.hpp:35-45)
    hamming_pairs(d)     hamming (simhash.hpp:47) over all i<j
    exact_pairs(tau)     cosine (ngram.hpp:184-202) over all i<j

Errors keep the reference's split (error.hpp:8-14): ValidationError for
caller-fixable input (exit code 2 in the reference CLI), RefsigRuntimeError
otherwise (exit 1). There is no CPU fallback: if the CUDA library or a device
is missing, construction fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Context", "ValidationError", "RefsigRuntimeError", "PairOverflowError", "WEIGHT_TF", "WEIGHT_TFIDF",
           "K3_AUTO", "K3_FP32", "K3_TENSOR", "library_path", "load_library", "split_keys"]

_HERE = os.path.dirname(os.path.abspath(__file__))
WEIGHT_TF = 0
WEIGHT_TFIDF = 1

OK, E_RUNTIME, E_VALIDATION, E_OVERFLOW = 0, 1, 2, 3
BUF_PAIRS, BUF_SIGNATURES, BUF_DF, BUF_FINGERPRINTS = 0, 1, 2, 3


class ValidationError(ValueError):
    """refsig::validation_error (reference error.hpp:11-14)."""


class RefsigRuntimeError(RuntimeError):
    """std::runtime_error class failures (CUDA errors, out of memory)."""


class PairOverflowError(RefsigRuntimeError):
    def __init__(self, msg, count):
        super().__init__(msg)
        self.count = count


def library_path() -> str:
    # REFSIG_GPU_LIB: another build of the same library (A/B measurement of kernel variants)
    return os.environ.get("REFSIG_GPU_LIB") or os.path.join(_HERE, "lib", "librefsig_gpu.so")


# Exported symbols and their ctypes signatures (tests check this list against
# include/refsig_gpu.h).
_P = ctypes.POINTER
_c = ctypes
SIGNATURES = {
    "refsig_gpu_create": ([_c.c_int, _P(_c.c_void_p)], _c.c_int),
    "refsig_gpu_destroy": ([_c.c_void_p], None),
    "refsig_gpu_last_error": ([_c.c_void_p], _c.c_char_p),
    "refsig_gpu_version": ([], _c.c_char_p),
    "refsig_gpu_set_stream": ([_c.c_void_p, _c.c_void_p], _c.c_int),
    "refsig_gpu_get_stream": ([_c.c_void_p], _c.c_void_p),
    "refsig_gpu_synchronize": ([_c.c_void_p], _c.c_int),
    "refsig_gpu_load_corpus": ([_c.c_void_p, _P(_c.c_uint32), _P(_c.c_uint64), _c.c_uint32, _c.c_uint32], _c.c_int),
    "refsig_gpu_load_corpus_device": ([_c.c_void_p, _c.c_void_p, _P(_c.c_uint64), _c.c_uint32, _c.c_uint32],
                                      _c.c_int),
    "refsig_gpu_count": ([_c.c_void_p, _c.c_int], _c.c_int),
    "refsig_gpu_get_counts": ([_c.c_void_p, _P(_c.c_uint64), _P(_c.c_uint32), _P(_c.c_uint32), _c.c_uint64,
                               _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_get_df": ([_c.c_void_p, _P(_c.c_uint32), _P(_c.c_float)], _c.c_int),
    "refsig_gpu_get_inv_norm": ([_c.c_void_p, _P(_c.c_float)], _c.c_int),
    "refsig_gpu_set_reference_docs": ([_c.c_void_p, _P(_c.c_uint32), _c.c_uint32], _c.c_int),
    "refsig_gpu_set_reference_vectors": ([_c.c_void_p, _c.c_uint32, _P(_c.c_uint64), _P(_c.c_uint32),
                                          _P(_c.c_float)], _c.c_int),
    "refsig_gpu_reference_union": ([_c.c_void_p, _P(_c.c_uint32)], _c.c_int),
    "refsig_gpu_sign": ([_c.c_void_p], _c.c_int),
    "refsig_gpu_get_signatures": ([_c.c_void_p, _P(_c.c_float)], _c.c_int),
    "refsig_gpu_mrc_pairs": ([_c.c_void_p, _c.c_float, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_simhash": ([_c.c_void_p, _c.c_uint64, _c.c_int, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_get_fingerprints": ([_c.c_void_p, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_hamming_pairs": ([_c.c_void_p, _c.c_int, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_exact_pairs": ([_c.c_void_p, _c.c_float, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_pair_cosines": ([_c.c_void_p, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_float)], _c.c_int),
    "refsig_gpu_attach_database": ([_c.c_void_p, _c.c_void_p], _c.c_int),
    "refsig_gpu_mrc_query_pairs": ([_c.c_void_p, _c.c_float, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_uint64)],
                                   _c.c_int),
    "refsig_gpu_hamming_query_pairs": ([_c.c_void_p, _c.c_int, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_uint64)],
                                       _c.c_int),
    "refsig_gpu_get_pairs": ([_c.c_void_p, _P(_c.c_uint64), _c.c_uint64], _c.c_int),
    "refsig_gpu_evaluate": ([_c.c_void_p, _c.c_uint32, _c.c_uint32, _c.c_void_p], _c.c_int),
    "refsig_gpu_get_corpus_freq": ([_c.c_void_p, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_get_signature_records": ([_c.c_void_p, _c.c_uint64, _P(_c.c_uint8), _c.c_uint64], _c.c_int),
    "refsig_gpu_get_pairs_csr16": ([_c.c_void_p, _c.c_uint32, _c.c_uint32, _P(_c.c_uint64), _P(_c.c_uint16),
                                    _c.c_uint64, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_set_global_df": ([_c.c_void_p, _P(_c.c_uint32), _c.c_uint32], _c.c_int),
    "refsig_gpu_set_reference_counts": ([_c.c_void_p, _c.c_uint32, _P(_c.c_uint64), _P(_c.c_uint32),
                                         _P(_c.c_uint32)], _c.c_int),
    "refsig_gpu_set_signatures": ([_c.c_void_p, _c.c_uint32, _c.c_uint32, _c.c_void_p, _c.c_int], _c.c_int),
    "refsig_gpu_load_text": ([_c.c_void_p, _P(_c.c_uint8), _P(_c.c_uint64), _c.c_uint32], _c.c_int),
    "refsig_gpu_simhash_text": ([_c.c_void_p], _c.c_int),
    "refsig_gpu_get_pairs_csr": ([_c.c_void_p, _c.c_uint32, _c.c_uint32, _P(_c.c_uint64), _P(_c.c_uint32), _c.c_uint64,
                                  _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_device_buffer": ([_c.c_void_p, _c.c_int, _P(_c.c_void_p), _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_mrc_pairs_rows": ([_c.c_void_p, _c.c_float, _c.c_uint32, _c.c_uint32, _P(_c.c_uint64), _c.c_uint64,
                                   _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_set_profiling": ([_c.c_void_p, _c.c_int], _c.c_int),
    "refsig_gpu_phase_times": ([_c.c_void_p, _P(_c.c_double), _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_launch_count": ([], _c.c_uint64),
    "refsig_gpu_mrc_step": ([_c.c_void_p, _c.c_int, _P(_c.c_uint32), _c.c_uint32, _c.c_float, _c.c_uint32, _c.c_uint32],
                            _c.c_int),
    "refsig_gpu_step_result": ([_c.c_void_p, _P(_c.c_uint64), _c.c_uint64, _P(_c.c_uint64)], _c.c_int),
    "refsig_gpu_set_k3_path": ([_c.c_void_p, _c.c_int], _c.c_int),
    "refsig_gpu_debug_check": ([_c.c_void_p], _c.c_int),
    "refsig_gpu_stage_corpus": ([_c.c_void_p, _P(_c.c_uint32), _P(_c.c_uint64), _c.c_uint32, _c.c_uint32], _c.c_int),
    "refsig_gpu_swap_corpus": ([_c.c_void_p], _c.c_int),
    "refsig_gpu_get_pairs_csr16_async": ([_c.c_void_p, _P(_c.c_uint64), _P(_c.c_uint16), _c.c_uint64, _P(_c.c_uint64)],
                                         _c.c_int),
    "refsig_gpu_wait_fetch": ([_c.c_void_p], _c.c_int),
}
K3_AUTO, K3_FP32, K3_TENSOR = 0, 1, 2
PHASES = ["count", "reference", "sign", "pair_tiles", "pair_emit", "simhash", "h2d", "d2h"]

_lib = None


def load_library():
    """Load librefsig_gpu.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        path = library_path()
        if not os.path.exists(path):
            raise RefsigRuntimeError(f"{path} not built: run __graft_entry__.build() / make")
        L = ctypes.CDLL(path)
        ab = bool(os.environ.get("REFSIG_GPU_LIB"))
        for name, (args, res) in SIGNATURES.items():
            if ab and not hasattr(L, name):  # an older build under A/B measurement
                continue
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _ptr(a, ct):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ct))


def split_keys(keys: np.ndarray):
    keys = np.asarray(keys, np.uint64)
    return (keys >> np.uint64(32)).astype(np.uint32), (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)


class Context:
    """One CUDA stream + device-resident corpus state (refsig_gpu_ctx)."""

    def __init__(self, device: int = 0):
        self._L = load_library()
        h = ctypes.c_void_p()
        rc = self._L.refsig_gpu_create(device, ctypes.byref(h))
        if rc != OK:
            raise RefsigRuntimeError(f"refsig_gpu_create(device={device}) failed with status {rc} "
                                     "(no usable sm_100a device)")
        self._h = h
        self.n_docs = 0
        self.vocab = 0
        self.K = 0

    # -- plumbing -------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._L.refsig_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def _check(self, rc, count=None):
        if rc == OK:
            return
        msg = self._L.refsig_gpu_last_error(self._h).decode()
        if rc == E_VALIDATION:
            raise ValidationError(msg)
        if rc == E_OVERFLOW:
            raise PairOverflowError(msg, count)
        raise RefsigRuntimeError(msg)

    def set_stream(self, stream_handle: int | None):
        self._check(self._L.refsig_gpu_set_stream(self._h, ctypes.c_void_p(stream_handle or 0)))

    @property
    def stream(self) -> int:
        return self._L.refsig_gpu_get_stream(self._h) or 0

    def synchronize(self):
        self._check(self._L.refsig_gpu_synchronize(self._h))

    # -- corpus / K1 ----------------------------------------------------------
    def load_corpus(self, tokens: np.ndarray, doc_off: np.ndarray, vocab: int):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        doc_off = np.ascontiguousarray(doc_off, np.uint64)
        if doc_off.ndim != 1 or len(doc_off) < 1:
            raise ValidationError("doc_off must hold n_docs+1 offsets")
        n = len(doc_off) - 1
        if n >= 1 and int(doc_off[-1]) > len(tokens):
            raise ValidationError("doc_off[-1] exceeds the token count")
        self._check(self._L.refsig_gpu_load_corpus(self._h, _ptr(tokens, ctypes.c_uint32),
                                                   _ptr(doc_off, ctypes.c_uint64), n, vocab))
        self._keep = tokens  # pinned/pageable source must outlive async copies
        self.n_docs, self.vocab = n, vocab

    def stage_corpus(self, tokens: np.ndarray, doc_off: np.ndarray, vocab: int):
        """Start the upload of the NEXT batch (copy stream; pinned tokens overlap
        with the current batch's compute). swap_corpus() makes it current."""
        tokens = np.ascontiguousarray(tokens, np.uint32)
        doc_off = np.ascontiguousarray(doc_off, np.uint64)
        n = len(doc_off) - 1
        if n >= 1 and int(doc_off[-1]) > len(tokens):
            raise ValidationError("doc_off[-1] exceeds the token count")
        self._check(self._L.refsig_gpu_stage_corpus(self._h, _ptr(tokens, ctypes.c_uint32),
                                                    _ptr(doc_off, ctypes.c_uint64), n, vocab))
        self._staged = (tokens, n, vocab)

    def swap_corpus(self):
        self._check(self._L.refsig_gpu_swap_corpus(self._h))
        tokens, n, vocab = self._staged
        self._keep = tokens
        self.n_docs, self.vocab = n, vocab

    def load_corpus_device(self, dev_ptr: int, doc_off: np.ndarray, vocab: int):
        """Tokens already in HBM (e.g. a torch uint32/int32 tensor's data_ptr())."""
        doc_off = np.ascontiguousarray(doc_off, np.uint64)
        n = len(doc_off) - 1
        self._check(self._L.refsig_gpu_load_corpus_device(self._h, ctypes.c_void_p(dev_ptr),
                                                          _ptr(doc_off, ctypes.c_uint64), n, vocab))
        self.n_docs, self.vocab = n, vocab

    def count(self, weighting: int = WEIGHT_TFIDF):
        self._check(self._L.refsig_gpu_count(self._h, weighting))

    def counts(self):
        """(rowptr, ids, counts): per doc the reference's NgramVector entries."""
        rowptr = np.zeros(self.n_docs + 1, np.uint64)
        nnz = ctypes.c_uint64()
        rc = self._L.refsig_gpu_get_counts(self._h, _ptr(rowptr, ctypes.c_uint64), None, None, 0, ctypes.byref(nnz))
        if rc not in (OK, E_OVERFLOW):
            self._check(rc)
        n = nnz.value
        ids = np.empty(max(n, 1), np.uint32)
        cnt = np.empty(max(n, 1), np.uint32)
        self._check(self._L.refsig_gpu_get_counts(self._h, _ptr(rowptr, ctypes.c_uint64), _ptr(ids, ctypes.c_uint32),
                                                  _ptr(cnt, ctypes.c_uint32), n, ctypes.byref(nnz)))
        return rowptr, ids[:n], cnt[:n]

    def corpus_freq(self) -> np.ndarray:
        """cf[vocab]: total occurrences of each term (SPEC FrequencyTable corpus_freq)."""
        cf = np.empty(self.vocab, np.uint64)
        self._check(self._L.refsig_gpu_get_corpus_freq(self._h, _ptr(cf, ctypes.c_uint64)))
        return cf

    def df(self):
        d = np.empty(self.vocab, np.uint32)
        idf = np.empty(self.vocab, np.float32)
        self._check(self._L.refsig_gpu_get_df(self._h, _ptr(d, ctypes.c_uint32), _ptr(idf, ctypes.c_float)))
        return d, idf

    def inv_norm(self):
        out = np.empty(self.n_docs, np.float32)
        self._check(self._L.refsig_gpu_get_inv_norm(self._h, _ptr(out, ctypes.c_float)))
        return out

    # -- reference / K2 -------------------------------------------------------
    def set_reference_docs(self, doc_ids):
        ids = np.ascontiguousarray(doc_ids, np.uint32)
        self._check(self._L.refsig_gpu_set_reference_docs(self._h, _ptr(ids, ctypes.c_uint32), len(ids)))
        self.K = len(ids)

    def set_reference_vectors(self, rowptr, term_ids, weights=None):
        rowptr = np.ascontiguousarray(rowptr, np.uint64)
        term_ids = np.ascontiguousarray(term_ids, np.uint32)
        w = None if weights is None else np.ascontiguousarray(weights, np.float32)
        K = len(rowptr) - 1
        self._check(self._L.refsig_gpu_set_reference_vectors(self._h, K, _ptr(rowptr, ctypes.c_uint64),
                                                             _ptr(term_ids, ctypes.c_uint32), _ptr(w, ctypes.c_float)))
        self.K = K

    def set_reference_partitions(self, parts):
        """Count-1 partition vectors (reference SPEC.md:306-314)."""
        rowptr = np.zeros(len(parts) + 1, np.uint64)
        rowptr[1:] = np.cumsum([len(p) for p in parts])
        ids = np.concatenate([np.asarray(p, np.uint32) for p in parts]) if parts else np.zeros(0, np.uint32)
        self.set_reference_vectors(rowptr, ids, None)

    def set_reference_counts(self, rowptr, term_ids, counts):
        """Reference vectors from (id, count) rows, weighted count * idf on the
        device like set_reference_docs (multi-GPU: the reference docs' rows
        come from the ranks that own them)."""
        rowptr = np.ascontiguousarray(rowptr, np.uint64)
        term_ids = np.ascontiguousarray(term_ids, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        K = len(rowptr) - 1
        self._check(self._L.refsig_gpu_set_reference_counts(self._h, K, _ptr(rowptr, ctypes.c_uint64),
                                                            _ptr(term_ids, ctypes.c_uint32),
                                                            _ptr(counts, ctypes.c_uint32)))
        self.K = K

    # -- multi-GPU building blocks (include/refsig_gpu.h) ----------------------
    def set_global_df(self, n_docs_global: int, df: np.ndarray | None = None):
        """idf from the global document frequencies: `df` from the host, or
        None when the device df buffer already holds the reduced table."""
        d = None if df is None else np.ascontiguousarray(df, np.uint32)
        if d is not None and len(d) != self.vocab:
            raise ValidationError("df must have vocab entries")
        self._check(self._L.refsig_gpu_set_global_df(self._h, _ptr(d, ctypes.c_uint32), int(n_docs_global)))

    def set_signatures(self, S, n_docs: int | None = None, K: int | None = None):
        """Install signatures for pair computations (a pairs-only context):
        `S` is a host float32 [n_docs, K] array or a device pointer (int)."""
        if isinstance(S, int):
            if n_docs is None or K is None:
                raise ValidationError("n_docs and K are required with a device pointer")
            self._check(self._L.refsig_gpu_set_signatures(self._h, int(n_docs), int(K), ctypes.c_void_p(S), 1))
        else:
            S = np.ascontiguousarray(S, np.float32)
            if S.ndim != 2:
                raise ValidationError("S must be [n_docs, K]")
            n_docs, K = S.shape
            self._check(self._L.refsig_gpu_set_signatures(self._h, n_docs, K, S.ctypes.data_as(ctypes.c_void_p), 0))
        self.n_docs, self.K = int(n_docs), int(K)

    def reference_union(self) -> int:
        u = ctypes.c_uint32()
        self._check(self._L.refsig_gpu_reference_union(self._h, ctypes.byref(u)))
        return u.value

    def sign(self, fetch: bool = True):
        self._check(self._L.refsig_gpu_sign(self._h))
        if not fetch:
            return None
        return self.signatures()

    def signatures(self):
        S = np.empty((self.n_docs, self.K), np.float32)
        self._check(self._L.refsig_gpu_get_signatures(self._h, _ptr(S, ctypes.c_float)))
        return S

    def signature_records(self, ref_id: int) -> np.ndarray:
        """uint8 [n_docs, 20 + 8K]: row d is the MRCS signature file of doc d
        (SPEC.md:401), written on the device."""
        rec = np.empty((self.n_docs, 20 + 8 * self.K), np.uint8)
        self._check(self._L.refsig_gpu_get_signature_records(self._h, ctypes.c_uint64(ref_id),
                                                             _ptr(rec, ctypes.c_uint8), rec.size))
        return rec

    # -- pairs ----------------------------------------------------------------
    def _pairs(self, fn, arg, out, fetch):
        n = ctypes.c_uint64()
        if out is not None:
            rc = fn(self._h, arg, _ptr(out, ctypes.c_uint64), len(out), ctypes.byref(n))
            self._check(rc, n.value)
            return out[: n.value]
        rc = fn(self._h, arg, None, 0, ctypes.byref(n))
        self._check(rc, n.value)
        if not fetch:
            return n.value
        keys = np.empty(n.value, np.uint64)
        if n.value:
            self._check(self._L.refsig_gpu_get_pairs(self._h, _ptr(keys, ctypes.c_uint64), n.value))
        return keys

    def pairs_csr(self, row_lo: int = 0, row_hi: int | None = None, rowptr: np.ndarray | None = None,
                  cols: np.ndarray | None = None):
        """The last pair call's pairs as CSR over rows [row_lo, row_hi):
        (rowptr[n+1] from 0, sorted column ids). Caller buffers (e.g. pinned)
        may be passed; cols must hold all pairs of the rows."""
        hi = self.n_docs if row_hi is None else row_hi
        n_rows = hi - row_lo
        if rowptr is None:
            rowptr = np.empty(n_rows + 1, np.uint64)
        n = ctypes.c_uint64()
        if cols is None:  # size query first (capacity 0: overflow status, exact count)
            rc = self._L.refsig_gpu_get_pairs_csr(self._h, row_lo, hi, _ptr(rowptr, ctypes.c_uint64), None, 0,
                                                  ctypes.byref(n))
            if rc != E_OVERFLOW:
                self._check(rc, n.value)
            cols = np.empty(max(n.value, 1), np.uint32)
        rc = self._L.refsig_gpu_get_pairs_csr(self._h, row_lo, hi, _ptr(rowptr, ctypes.c_uint64),
                                              _ptr(cols, ctypes.c_uint32), len(cols), ctypes.byref(n))
        self._check(rc, n.value)
        return rowptr[: n_rows + 1], cols[: n.value]

    def pairs_csr16(self, row_lo: int = 0, row_hi: int | None = None, rowptr: np.ndarray | None = None,
                    cols: np.ndarray | None = None):
        """pairs_csr with uint16 column ids (n_docs <= 65536): half the bytes."""
        hi = self.n_docs if row_hi is None else row_hi
        n_rows = hi - row_lo
        if rowptr is None:
            rowptr = np.empty(n_rows + 1, np.uint64)
        n = ctypes.c_uint64()
        if cols is None:
            rc = self._L.refsig_gpu_get_pairs_csr16(self._h, row_lo, hi, _ptr(rowptr, ctypes.c_uint64), None, 0,
                                                    ctypes.byref(n))
            if rc != E_OVERFLOW:
                self._check(rc, n.value)
            cols = np.empty(max(n.value, 1), np.uint16)
        rc = self._L.refsig_gpu_get_pairs_csr16(self._h, row_lo, hi, _ptr(rowptr, ctypes.c_uint64),
                                                _ptr(cols, ctypes.c_uint16), len(cols), ctypes.byref(n))
        self._check(rc, n.value)
        return rowptr[: n_rows + 1], cols[: n.value]

    def pairs_csr16_async(self, rowptr: np.ndarray, cols: np.ndarray) -> int:
        """Start copying the last pair call's CSR (uint16 columns) into the given
        pinned host arrays; returns the exact count at once. wait_fetch() completes it."""
        n = ctypes.c_uint64()
        rc = self._L.refsig_gpu_get_pairs_csr16_async(self._h, _ptr(rowptr, ctypes.c_uint64),
                                                      _ptr(cols, ctypes.c_uint16), len(cols), ctypes.byref(n))
        self._check(rc, n.value)
        return n.value

    def wait_fetch(self):
        self._check(self._L.refsig_gpu_wait_fetch(self._h))

    def mrc_pairs(self, tau: float, out: np.ndarray | None = None, fetch: bool = True):
        """Sorted keys (i<<32|j) of all i<j with compare(S_i,S_j) >= tau."""
        return self._pairs(self._L.refsig_gpu_mrc_pairs, ctypes.c_float(tau), out, fetch)

    def mrc_pairs_rows(self, tau: float, row_lo: int, row_hi: int, out: np.ndarray | None = None,
                       fetch: bool = True):
        """Pairs i<j with row_lo <= i < row_hi (a rank's shard of the triangle)."""
        n = ctypes.c_uint64()
        if out is not None:
            rc = self._L.refsig_gpu_mrc_pairs_rows(self._h, ctypes.c_float(tau), row_lo, row_hi,
                                                   _ptr(out, ctypes.c_uint64), len(out), ctypes.byref(n))
            self._check(rc, n.value)
            return out[: n.value]
        rc = self._L.refsig_gpu_mrc_pairs_rows(self._h, ctypes.c_float(tau), row_lo, row_hi, None, 0,
                                               ctypes.byref(n))
        self._check(rc, n.value)
        if not fetch:
            return n.value
        keys = np.empty(n.value, np.uint64)
        if n.value:
            self._check(self._L.refsig_gpu_get_pairs(self._h, _ptr(keys, ctypes.c_uint64), n.value))
        return keys

    def mrc_step(self, ref_doc_ids, tau: float, weighting: int = WEIGHT_TFIDF, row_lo: int = 0,
                 row_hi: int | None = None):
        """count -> reference -> sign -> pairs, enqueued as one CUDA-graph replay
        after the first call; collect with step_result()."""
        ids = np.ascontiguousarray(ref_doc_ids, np.uint32)
        hi = self.n_docs if row_hi is None else row_hi
        self._check(self._L.refsig_gpu_mrc_step(self._h, weighting, _ptr(ids, ctypes.c_uint32), len(ids),
                                                ctypes.c_float(tau), row_lo, hi))
        self.K = len(ids)

    def step_result(self, out: np.ndarray | None = None, fetch: bool = False):
        n = ctypes.c_uint64()
        if out is not None:
            rc = self._L.refsig_gpu_step_result(self._h, _ptr(out, ctypes.c_uint64), len(out), ctypes.byref(n))
            self._check(rc, n.value)
            return out[: n.value]
        self._check(self._L.refsig_gpu_step_result(self._h, None, 0, ctypes.byref(n)), n.value)
        if not fetch:
            return n.value
        keys = np.empty(n.value, np.uint64)
        if n.value:
            self._check(self._L.refsig_gpu_get_pairs(self._h, _ptr(keys, ctypes.c_uint64), n.value))
        return keys

    def set_k3_path(self, path: int):
        """K3_AUTO / K3_FP32 (CUDA cores) / K3_TENSOR (tcgen05) for the pair calls."""
        self._check(self._L.refsig_gpu_set_k3_path(self._h, int(path)))

    def debug_check(self):
        """With REFSIG_CANARY=1: raise if a kernel wrote past any device buffer."""
        self._check(self._L.refsig_gpu_debug_check(self._h))

    # -- measurement ----------------------------------------------------------
    def set_profiling(self, on: bool):
        self._check(self._L.refsig_gpu_set_profiling(self._h, 1 if on else 0))

    def phase_times(self) -> dict:
        """{phase: (total_ms, calls)} since set_profiling (events on this stream)."""
        ms = (ctypes.c_double * len(PHASES))()
        calls = (ctypes.c_uint64 * len(PHASES))()
        self._check(self._L.refsig_gpu_phase_times(self._h, ms, calls))
        return {p: (ms[i], calls[i]) for i, p in enumerate(PHASES)}

    @staticmethod
    def launch_count() -> int:
        return load_library().refsig_gpu_launch_count()

    def evaluate(self, row_lo: int = 0, row_hi: int | None = None) -> dict:
        """SPEC eval (Eq. 2/3) over all pairs i<j, row_lo <= i < row_hi: MAE,
        mean error and variance of MRC (and Simhash, if fingerprints exist)
        against the exact cosine, fused on the GPU."""
        class _Eval(ctypes.Structure):
            _fields_ = [("pairs", ctypes.c_uint64)] + [(k, ctypes.c_double) for k in (
                "mrc_mae", "mrc_mean_error", "mrc_variance", "simhash_mae", "simhash_mean_error",
                "simhash_variance")]
        e = _Eval()
        hi = self.n_docs if row_hi is None else row_hi
        self._check(self._L.refsig_gpu_evaluate(self._h, row_lo, hi, ctypes.byref(e)))
        return {k: getattr(e, k) for k, _ in _Eval._fields_}

    def load_text(self, text, byte_off: np.ndarray):
        """Raw documents text[byte_off[d]:byte_off[d+1]] (bytes or uint8 array):
        the corpus becomes their character 3-grams (vocab 17576)."""
        t = np.frombuffer(text, np.uint8) if isinstance(text, (bytes, bytearray)) else np.ascontiguousarray(text, np.uint8)
        off = np.ascontiguousarray(byte_off, np.uint64)
        if len(off) < 2 or int(off[-1]) > len(t):
            raise ValidationError("byte_off must have n_docs+1 entries within the text")
        if len(t) == 0:
            t = np.zeros(1, np.uint8)
        self._check(self._L.refsig_gpu_load_text(self._h, _ptr(t, ctypes.c_uint8), _ptr(off, ctypes.c_uint64),
                                                 len(off) - 1))
        self.n_docs = len(off) - 1
        self.vocab = 26 ** 3

    def simhash_text(self, fetch: bool = True):
        """Per-document simhash of the loaded text's words (MD5, +-1 votes)."""
        self._check(self._L.refsig_gpu_simhash_text(self._h))
        return self.fingerprints() if fetch else None

    def simhash(self, seed: int = 0, weighting: int = WEIGHT_TFIDF, term_hash: np.ndarray | None = None,
                fetch: bool = True):
        th = None if term_hash is None else np.ascontiguousarray(term_hash, np.uint64)
        self._check(self._L.refsig_gpu_simhash(self._h, seed, weighting, _ptr(th, ctypes.c_uint64)))
        if not fetch:
            return None
        return self.fingerprints()

    def fingerprints(self):
        fp = np.empty(self.n_docs, np.uint64)
        self._check(self._L.refsig_gpu_get_fingerprints(self._h, _ptr(fp, ctypes.c_uint64)))
        return fp

    def hamming_pairs(self, max_dist: int = 3, out=None, fetch: bool = True):
        return self._pairs(self._L.refsig_gpu_hamming_pairs, max_dist, out, fetch)

    def exact_pairs(self, tau_cos: float, out=None, fetch: bool = True):
        return self._pairs(self._L.refsig_gpu_exact_pairs, ctypes.c_float(tau_cos), out, fetch)

    def pair_cosines(self, keys: np.ndarray) -> np.ndarray:
        keys = np.ascontiguousarray(keys, np.uint64)
        out = np.empty(len(keys), np.float32)
        self._check(self._L.refsig_gpu_pair_cosines(self._h, _ptr(keys, ctypes.c_uint64), len(keys),
                                                    _ptr(out, ctypes.c_float)))
        return out

    # -- query-vs-database ----------------------------------------------------
    def attach_database(self, db: "Context"):
        self._check(self._L.refsig_gpu_attach_database(self._h, db.handle))
        self.K = db.K
        self._db = db

    def mrc_query_pairs(self, tau: float, out=None, fetch: bool = True):
        return self._pairs(self._L.refsig_gpu_mrc_query_pairs, ctypes.c_float(tau), out, fetch)

    def hamming_query_pairs(self, max_dist: int = 3, out=None, fetch: bool = True):
        return self._pairs(self._L.refsig_gpu_hamming_query_pairs, max_dist, out, fetch)

    def device_buffer(self, which: int):
        p = ctypes.c_void_p()
        n = ctypes.c_uint64()
        self._check(self._L.refsig_gpu_device_buffer(self._h, which, ctypes.byref(p), ctypes.byref(n)))
        return p.value or 0, n.value
