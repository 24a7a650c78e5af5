"""Sharded K1/K2 emulated on one GPU: W document shards, each
in its own context, exchange df (sum) and signatures (rank-ordered concat)
through shard.LocalComm; the signatures and the MRC candidate list must be
bit-identical to the single-context step (same global df, same reference
weighting kernel, same unit-signature arithmetic)."""
import numpy as np
import pytest

import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
from paper_1810_03099_b200 import shard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_step_matches_single_gpu(gpu_ctx_factory, world):
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(6000)
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    tau = 0.95
    one = gpu_ctx_factory()
    one.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    one.count(R.WEIGHT_TFIDF)
    one.set_reference_docs(refs)
    S_one = one.sign()
    keys_one = one.mrc_pairs(tau)

    shards = shard.doc_shards(cp.doc_off, world)
    ctxs = [gpu_ctx_factory() for _ in shards]
    ref_ctx = gpu_ctx_factory()
    comm = shard.LocalComm()
    for c, (lo, hi) in zip(ctxs, shards):
        t, o = shard.shard_corpus(cp.tokens, cp.doc_off, lo, hi)
        c.load_corpus(t, o, cp.vocab)
        c.count(R.WEIGHT_TFIDF)
    df = comm.allreduce_df(ctxs)
    assert np.array_equal(df, one.df()[0])
    rp, ids, cnt = shard.reference_rows(ref_ctx, cp.tokens, cp.doc_off, refs, cp.vocab)
    for c in ctxs:
        c.set_global_df(cp.n_docs, df)
        c.set_reference_counts(rp, ids, cnt)
        c.sign(fetch=False)
    S_all = comm.allgather_signatures(ctxs)
    assert S_all.tobytes() == S_one.tobytes()  # bit-identical signatures

    pairs = gpu_ctx_factory()
    pairs.set_signatures(S_all)
    parts = [pairs.mrc_pairs_rows(tau, lo, hi).copy() for lo, hi in shard.row_shards(cp.n_docs, world)]
    keys = np.concatenate(parts)
    assert np.array_equal(keys, keys_one)


def test_set_signatures_from_device_pointer_and_in_place_df(gpu_ctx_factory):
    import torch
    cp, cfg = C.config_corpus("c0")
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count(R.WEIGHT_TFIDF)
    df0, idf0 = ctx.df()
    ctx.set_global_df(cp.n_docs)  # device df already global: same table
    assert np.array_equal(ctx.df()[1], idf0)
    ctx.set_global_df(2 * cp.n_docs)  # a larger corpus changes the idf
    assert not np.array_equal(ctx.df()[1], idf0)
    ctx.set_global_df(cp.n_docs, df0)
    ctx.set_reference_docs(refs)
    S = ctx.sign()
    keys = ctx.mrc_pairs(0.9)
    dev = torch.from_numpy(S).cuda()
    pairs = gpu_ctx_factory()
    pairs.set_signatures(dev.data_ptr(), *S.shape)
    assert np.array_equal(pairs.mrc_pairs(0.9), keys)
    with pytest.raises(R.ValidationError, match="no corpus loaded"):
        pairs.count()  # a pairs-only context has no corpus
