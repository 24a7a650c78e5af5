"""Multi-rank host logic on CPU (gloo, world size 2): the triangle row-panel
sharding used by bench.py --gpus N. Each rank computes its
rows' MRC/Hamming pairs (the oracle stands in for the GPU kernel here), the
rank-ordered concatenation must equal the single-rank result, and the
max-over-ranks timing reduction works."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1810_03099_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_shards_cover_triangle_once():
    for n in [1, 127, 128, 129, 2000, 18846]:
        for w in [1, 2, 3, 4, 8]:
            sh = shard.row_shards(n, w)
            assert len(sh) == w and sh[0][0] == 0 and sh[-1][1] == n
            for (a, b), (c, d) in zip(sh, sh[1:]):
                assert b == c and a <= b
            assert all(lo % 128 == 0 or lo == hi == n for lo, hi in sh)
            assert sum(shard.pairs_in_rows(n, lo, hi) for lo, hi in sh) == n * (n - 1) // 2


def test_row_shards_balanced():
    sh = shard.row_shards(18846, 8)
    tiles = shard.panel_tiles(18846)
    per = [sum(tiles[lo // 128:(hi + 127) // 128]) for lo, hi in sh]
    assert max(per) / (sum(per) / 8) < 1.1  # 128-row panel granularity


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1810_03099_b200 import corpus as C
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cp, cfg = C.config_corpus("c0")
    cp = cp.slice_docs(600)
    refs = C.sample_refs(0, cp.n_docs, 10)
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
    lo, hi = shard.row_shards(cp.n_docs, world)[rank]
    mine, _ = oracle.mrc_pairs(o.S, 0.95, 1e-5, lo, hi, threads=1)
    keys = shard.gather_sorted_keys(mine, world, dist.all_gather_object)
    fp = oracle.simhash(o.counts, o.idf, 0, threads=1)
    hk = shard.gather_sorted_keys(oracle.hamming_pairs(fp, 20, lo, hi, threads=1), world, dist.all_gather_object)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full, _ = oracle.mrc_pairs(o.S, 0.95, 1e-5, threads=1)
        fullh = oracle.hamming_pairs(fp, 20, threads=1)
        q.put((bool(np.array_equal(keys, full)), bool(np.array_equal(hk, fullh)), len(full), t.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_pairs_equal_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    same_mrc, same_ham, n, tmax = res
    assert same_mrc and same_ham and n > 0
    assert tmax == 2.0


class _FakeShardCtx:
    """The two calls TorchComm's gloo path makes on a context."""

    def __init__(self, df, S):
        self._df, self._S = df, S

    def df(self):
        return self._df, None

    def signatures(self):
        return self._S


def _comm_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    n_local = [5, 3][rank]
    ctx = _FakeShardCtx(rng.integers(0, 9, 50).astype(np.uint32), rng.random((n_local, 4)).astype(np.float32))
    comm = shard.TorchComm(dist)
    df = comm.allreduce_df(ctx)
    S, counts = comm.allgather_signatures(ctx, n_local, 4, 5)
    q.put((rank, df, S, counts))
    dist.destroy_process_group()


def test_torch_comm_gloo_df_sum_and_ordered_signatures():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    ref_df = sum(np.random.default_rng(r).integers(0, 9, 50) for r in range(world))
    # each fake context draws df, then S, from its rank's generator
    ref_S = []
    for r, n in zip(range(world), [5, 3]):
        g = np.random.default_rng(r)
        g.integers(0, 9, 50)
        ref_S.append(g.random((n, 4)).astype(np.float32))
    ref_S = np.concatenate(ref_S)
    for rank, df, S, counts in res:
        assert np.array_equal(df, ref_df.astype(np.uint32))
        assert counts == [5, 3]
        assert S.tobytes() == ref_S.tobytes()


def test_doc_shards_cover_and_balance():
    from paper_1810_03099_b200 import corpus as C
    cp, _ = C.config_corpus("c0")
    for w in [1, 2, 3, 8]:
        sh = shard.doc_shards(cp.doc_off, w)
        assert sh[0][0] == 0 and sh[-1][1] == cp.n_docs and all(b == c for (_, b), (c, _) in zip(sh, sh[1:]))
        toks = [int(cp.doc_off[hi]) - int(cp.doc_off[lo]) for lo, hi in sh]
        assert max(toks) <= sum(toks) / w * 1.1 + 5000


def _weak_worker(rank, world, port, q):
    """bench.py --gpus N (weak scaling): rank r runs its own batch, a seeded
    document permutation of the corpus; the helpers reduce over ranks."""
    import torch.distributed as dist

    import bench
    import oracle
    from paper_1810_03099_b200 import corpus as C
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cp, _ = C.config_corpus("c0")
    cp = cp.slice_docs(500)
    refs = C.sample_refs(0, cp.n_docs, 10)
    tok, off, rrefs = bench.permuted_batches(cp, refs, 1, seed=1000 + rank)[0]
    o = oracle.mrc_pipeline(np.asarray(tok), off, cp.vocab, rrefs)
    pairs, _ = oracle.mrc_pairs(o.S, 0.95, 1e-5, threads=1)
    # map the batch's pairs back to original document ids: the same set as the unpermuted corpus
    lens = np.diff(cp.doc_off).astype(np.int64)
    perm = np.empty(cp.n_docs, np.int64)
    # the batch's permutation (bench.permuted_batches draws it from the same seed): document p of
    # the batch is original document perm[p]
    rng = np.random.default_rng(1000 + rank)
    perm[:] = rng.permutation(cp.n_docs)
    assert np.array_equal(np.diff(off).astype(np.int64), lens[perm])
    i = perm[(pairs >> np.uint64(32)).astype(np.int64)]
    j = perm[(pairs & np.uint64(0xFFFFFFFF)).astype(np.int64)]
    orig = np.sort((np.minimum(i, j).astype(np.uint64) << np.uint64(32)) | np.maximum(i, j).astype(np.uint64))
    mx = bench.allreduce(dist, [float(rank + 1), 7.0], None, "max")
    sm = bench.allreduce(dist, [float(len(pairs))], None, "sum")
    if rank == 0:
        o0 = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
        ref_pairs, _ = oracle.mrc_pairs(o0.S, 0.95, 1e-5, threads=1)
        q.put((orig.tobytes(), ref_pairs.tobytes(), mx, sm, len(ref_pairs)))
    else:
        q.put((orig.tobytes(), None, mx, sm, None))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_weak_scaling_batches():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_weak_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = next(r for r in res if r[1] is not None)
    for orig, _, mx, sm, _ in res:
        assert orig == ref[1]  # every rank's batch is the same work (same pair set up to the permutation)
        assert mx == [2.0, 7.0] and sm == [2.0 * ref[4]]
