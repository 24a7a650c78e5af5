"""GPU: the captured MRC step (refsig_gpu_mrc_step, CUDA-graph replay) gives
the same sorted candidates as the call-by-call API, across replays, changed
references, changed tau, row shards and a reloaded corpus."""
import numpy as np
import pytest

import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C

pytestmark = pytest.mark.gpu


def eager(ctx, refs, tau, lo=0, hi=None):
    ctx.count()
    ctx.set_reference_docs(refs)
    ctx.sign(fetch=False)
    return ctx.mrc_pairs_rows(tau, lo, ctx.n_docs if hi is None else hi)


def test_step_replays_match_eager(gpu_ctx_factory):
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(6000)
    refs = C.sample_refs(0, cp.n_docs, 20)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    want = eager(ctx, refs, 0.99)
    for _ in range(4):  # first call eager + capture, then graph replays
        ctx.mrc_step(refs, 0.99)
        got = ctx.step_result(fetch=True)
        assert np.array_equal(got, want)
    # signatures are those of the step
    assert np.allclose(ctx.signatures(), (eager(ctx, refs, 0.99), ctx.signatures())[1])
    # other references / tau / rows re-capture
    refs2 = C.sample_refs(5, cp.n_docs, 20)
    want2 = eager(ctx, refs2, 0.95, 128, 2048)
    for _ in range(2):
        ctx.mrc_step(refs2, 0.95, R.WEIGHT_TFIDF, 128, 2048)
        assert np.array_equal(ctx.step_result(fetch=True), want2)
    ctx.mrc_step(refs, 0.99)
    out = np.empty(len(want) + 5, np.uint64)
    got = ctx.step_result(out=out)
    assert np.array_equal(got, want)


def test_step_after_reload_and_growth(gpu_ctx_factory):
    cp, cfg = C.config_corpus("c0")
    refs = C.sample_refs(0, 1000, 10)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens[: int(cp.doc_off[1000])], cp.doc_off[:1001], cp.vocab)
    ctx.mrc_step(refs, 0.999)
    a = ctx.step_result(fetch=True)
    ctx.mrc_step(refs, 0.999)
    assert np.array_equal(ctx.step_result(fetch=True), a)
    # a larger corpus (new buffers) and a low tau (many candidates: buffer growth)
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    want = eager(ctx, refs, 0.5)
    for _ in range(3):
        ctx.mrc_step(refs, 0.5)
        assert np.array_equal(ctx.step_result(fetch=True), want)


def test_step_requires_collect(gpu_ctx_factory):
    cp, _ = C.config_corpus("c0")
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    refs = C.sample_refs(0, cp.n_docs, 10)
    ctx.mrc_step(refs, 0.99)
    with pytest.raises(R.ValidationError):
        ctx.mrc_step(refs, 0.99)
    ctx.step_result()


def test_same_layout_reload_keeps_step_graph_but_reads_new_tokens(gpu_ctx_factory):
    """A batch with the same doc_off reuses the work plan and the captured
    step graph; the graph must read the newly uploaded tokens."""
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(3000)
    refs = C.sample_refs(0, cp.n_docs, 20)
    rng = np.random.default_rng(3)
    tok2 = cp.tokens.copy()
    flip = rng.random(len(tok2)) < 0.3
    tok2[flip] = rng.integers(0, cp.vocab, int(flip.sum()), dtype=np.uint32)
    fresh = gpu_ctx_factory()
    fresh.load_corpus(tok2, cp.doc_off, cp.vocab)
    want2 = eager(fresh, refs, 0.95)
    fresh.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    want1 = eager(fresh, refs, 0.95)
    assert not np.array_equal(want1, want2)
    ctx = gpu_ctx_factory()
    for tok, want in [(cp.tokens, want1), (tok2, want2), (cp.tokens, want1), (tok2, want2)]:
        ctx.load_corpus(tok, cp.doc_off, cp.vocab)
        ctx.mrc_step(refs, 0.95)
        assert np.array_equal(ctx.step_result(fetch=True), want)
        rowptr, ids, counts = ctx.counts()  # counted rows are the new batch's
        assert int(rowptr[-1]) == int(fresh_counts_total(tok, cp))


def fresh_counts_total(tok, cp):
    import oracle
    return len(oracle.count(tok, cp.doc_off).ids)


@pytest.mark.parametrize("K", [10, 41, 64])
def test_step_tensor_core_and_cuda_core_k3(gpu_ctx_factory, K):
    """The captured step with K3 on tcgen05 (K <= 41) and on CUDA cores (K = 64)."""
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(2500)
    refs = C.sample_refs(2, cp.n_docs, K)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    want = eager(ctx, refs, 0.9)
    for _ in range(3):
        ctx.mrc_step(refs, 0.9)
        assert np.array_equal(ctx.step_result(fetch=True), want)


@pytest.mark.parametrize("K", [64, 128])
def test_step_large_k_graph(gpu_ctx_factory, K):
    """The captured step with the chunked tcgen05 K3 (K' = 208 / 400) and the
    PDL chain (reference build, sign, forms) equals the eager calls."""
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(3000)
    refs = C.sample_refs(3, cp.n_docs, K)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    want = eager(ctx, refs, 0.99)
    for _ in range(3):
        ctx.mrc_step(refs, 0.99)
        assert np.array_equal(ctx.step_result(fetch=True), want)
    assert ctx.reference_union() > 0
