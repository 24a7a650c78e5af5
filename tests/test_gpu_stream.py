"""Streaming batches (stage_corpus / swap_corpus: the next batch's upload on a
copy stream while the current one computes) give exactly what load_corpus
gives, batch after batch; and the query join's cached database column forms
(built once per database signature) give what a fresh context gives."""
import numpy as np
import pytest

import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C

pytestmark = pytest.mark.gpu


def _batches(n_batches=3, n=700):
    cp, _ = C.config_corpus("c0")
    out = []
    for b in range(n_batches):  # different document subsets and layouts
        lo = b * 400
        sub = cp.slice_docs(lo + n)
        off = (sub.doc_off[lo:] - sub.doc_off[lo]).astype(np.uint64)
        tok = sub.tokens[int(sub.doc_off[lo]):int(sub.doc_off[-1])]
        out.append((np.ascontiguousarray(tok), off, cp.vocab))
    return out


def test_stage_swap_equals_load(gpu_ctx_factory):
    batches = _batches()
    refs = np.arange(10, dtype=np.uint32) * 7
    a, b = gpu_ctx_factory(), gpu_ctx_factory()
    b.stage_corpus(*batches[0])
    for k, (tok, off, V) in enumerate(batches):
        b.swap_corpus()
        if k + 1 < len(batches):
            b.stage_corpus(*batches[k + 1])  # in flight while batch k computes
        b.count()
        b.set_reference_docs(refs)
        Sb = b.sign()
        kb = b.mrc_pairs(0.95)
        a.load_corpus(tok, off, V)
        a.count()
        a.set_reference_docs(refs)
        Sa = a.sign()
        ka = a.mrc_pairs(0.95)
        assert np.array_equal(Sa, Sb) and np.array_equal(ka, kb), f"batch {k}"


def test_stage_two_ahead_equals_load(gpu_ctx_factory):
    """Two batches staged ahead (the copy engine always has the next upload
    queued): each batch still gives what load_corpus gives; a third stage
    before a swap is refused."""
    batches = _batches(4)
    refs = np.arange(10, dtype=np.uint32) * 7
    a, b = gpu_ctx_factory(), gpu_ctx_factory()
    b.stage_corpus(*batches[0])
    b.stage_corpus(*batches[1])
    with pytest.raises((R.ValidationError, R.RefsigRuntimeError)):
        b.stage_corpus(*batches[2])
    for k, (tok, off, V) in enumerate(batches):
        b.swap_corpus()
        b.count()
        b.set_reference_docs(refs)
        Sb = b.sign()
        if k + 2 < len(batches):
            b.stage_corpus(*batches[k + 2])
        kb = b.mrc_pairs(0.95)
        a.load_corpus(tok, off, V)
        a.count()
        a.set_reference_docs(refs)
        Sa = a.sign()
        ka = a.mrc_pairs(0.95)
        assert np.array_equal(Sa, Sb) and np.array_equal(ka, kb), f"batch {k}"


def test_query_join_cached_database_forms(gpu_ctx_factory):
    cp, _ = C.config_corpus("c0")
    refs = C.sample_refs(0, cp.n_docs, 64)
    db = gpu_ctx_factory()
    db.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    db.count()
    db.set_reference_docs(refs)
    db.sign(fetch=False)
    q = gpu_ctx_factory()
    q.attach_database(db)
    results = []
    for tau in (0.9, 0.99, 0.9):  # second and third calls reuse the database forms
        q.load_corpus(cp.tokens[: int(cp.doc_off[300])], cp.doc_off[:301], cp.vocab)
        q.count()
        q.sign(fetch=False)
        results.append(q.mrc_query_pairs(tau))
    assert np.array_equal(results[0], results[2])
    fresh = gpu_ctx_factory()
    fresh.attach_database(db)
    fresh.load_corpus(cp.tokens[: int(cp.doc_off[300])], cp.doc_off[:301], cp.vocab)
    fresh.count()
    fresh.sign(fetch=False)
    assert np.array_equal(fresh.mrc_query_pairs(0.99), results[1])
    # re-signing the database with another reference invalidates the cache
    db.set_reference_docs(C.sample_refs(1, cp.n_docs, 64))
    db.sign(fetch=False)
    q.load_corpus(cp.tokens[: int(cp.doc_off[300])], cp.doc_off[:301], cp.vocab)
    q.count()
    q.sign(fetch=False)
    k_new = q.mrc_query_pairs(0.99)
    ref = gpu_ctx_factory()
    ref.attach_database(db)
    ref.load_corpus(cp.tokens[: int(cp.doc_off[300])], cp.doc_off[:301], cp.vocab)
    ref.count()
    ref.sign(fetch=False)
    assert np.array_equal(ref.mrc_query_pairs(0.99), k_new)


def test_async_csr16_fetch_equals_sync(gpu_ctx_factory):
    """get_pairs_csr16_async (two slots in flight) delivers what get_pairs_csr16 does."""
    import torch
    batches = _batches(4, 600)
    refs = np.arange(10, dtype=np.uint32) * 5
    ctx = gpu_ctx_factory()
    host = [(torch.empty(601, dtype=torch.int64).pin_memory().numpy().view(np.uint64),
             torch.empty(200_000, dtype=torch.int16).pin_memory().numpy().view(np.uint16)) for _ in range(2)]
    want, got = [], []
    for k, (tok, off, V) in enumerate(batches):
        ctx.load_corpus(tok, off, V)
        ctx.count()
        ctx.set_reference_docs(refs)
        ctx.sign(fetch=False)
        ctx.mrc_pairs_rows(0.9, 0, len(off) - 1, fetch=False)
        want.append(ctx.pairs_csr16())
        ctx.wait_fetch()
        if k >= 2:
            rp, cs = host[k & 1]
            got.append((rp.copy(), cs[: int(rp[-1])].copy()))  # slot reused: batch k-2 complete
        n = ctx.pairs_csr16_async(*host[k & 1])
        assert n == len(want[-1][1])
    ctx.wait_fetch()
    for k in (2, 3):
        rp, cs = host[k & 1]
        got.append((rp.copy(), cs[: int(rp[-1])].copy()))
    # got holds batches 0,1 (read when their slots were reused) then 2,3
    for (wr, wc), (gr, gc) in zip(want, got):
        assert np.array_equal(wr, gr) and np.array_equal(wc, gc)


def _ragged(V, n_docs=300, seed=1):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 900, n_docs)  # ragged: empty documents, T not a multiple of 32
    off = np.zeros(n_docs + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    tok = (rng.zipf(1.3, int(off[-1])) * 2654435761 % V).astype(np.uint32)
    tok[: min(len(tok), 50)] = V - 1  # the widest id of the vocabulary
    return tok, off


@pytest.mark.parametrize("V", [30000, 65537, 130000, 1 << 20, (1 << 24) + 1])
def test_stage_equals_load_vocab_widths(gpu_ctx_factory, V):
    """A staged batch counts exactly like load_corpus at every id width."""
    tok, off = _ragged(V)
    a, b = gpu_ctx_factory(), gpu_ctx_factory()
    b.stage_corpus(tok, off, V)
    b.swap_corpus()
    b.count()
    a.load_corpus(tok, off, V)
    a.count()
    for x, y in zip(a.counts(), b.counts()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("bad", [130001, 1 << 31])
def test_stage_out_of_vocab(gpu_ctx_factory, bad):
    """An id >= vocab in a staged batch is reported like in a loaded one."""
    V = 130000
    tok, off = _ragged(V)
    tok[len(tok) // 2] = bad
    b = gpu_ctx_factory()
    b.stage_corpus(tok, off, V)
    b.swap_corpus()
    b.count()
    with pytest.raises(R.ValidationError, match="vocab"):
        b.synchronize()
