"""GPU: the rank shards of the pair triangle (mrc_pairs_rows over
shard.row_shards) concatenate to exactly the single-call result — the
property bench.py --gpus N relies on. One GPU, sequential calls."""
import numpy as np
import pytest

import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
from paper_1810_03099_b200 import shard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_concatenate_to_full(gpu_ctx_factory, world):
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(5000)
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(C.sample_refs(0, cp.n_docs, 20))
    ctx.sign(fetch=False)
    full = ctx.mrc_pairs(0.99)
    parts = [ctx.mrc_pairs_rows(0.99, lo, hi) for lo, hi in shard.row_shards(cp.n_docs, world)]
    assert np.array_equal(np.concatenate(parts), full)


def test_row_range_validation(gpu_ctx_factory):
    cp, _ = C.config_corpus("c0")
    ctx = gpu_ctx_factory()
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(C.sample_refs(0, cp.n_docs, 10))
    ctx.sign(fetch=False)
    with pytest.raises(R.ValidationError):
        ctx.mrc_pairs_rows(0.9, 5, 300)  # not tile aligned
    assert len(ctx.mrc_pairs_rows(0.9, cp.n_docs, cp.n_docs)) == 0  # empty shard
