"""Sharding of the all-pairs triangle across ranks.

The i<j triangle is cut into contiguous 128-row panels; panel p holds
nb - p tiles of 128x128 pairs. Ranks get contiguous panel ranges with about
equal tile counts, so the concatenation of the ranks' sorted key lists (rank
order) is the globally sorted candidate list and no pair is computed twice.
"""
from __future__ import annotations

TILE = 128


def panel_tiles(n_docs: int) -> list[int]:
    nb = -(-n_docs // TILE)
    return [nb - p for p in range(nb)]


def row_shards(n_docs: int, world: int) -> list[tuple[int, int]]:
    """[(row_lo, row_hi)] per rank; row_lo is 128-aligned, row_hi is aligned or n_docs."""
    if world < 1:
        raise ValueError("world must be >= 1")
    tiles = panel_tiles(n_docs)
    nb = len(tiles)
    total = sum(tiles)
    bounds = [0]
    acc = 0
    p = 0
    for r in range(1, world):
        target = total * r / world
        while p < nb and acc + tiles[p] / 2 < target:
            acc += tiles[p]
            p += 1
        bounds.append(max(p, bounds[-1]))
    bounds.append(nb)
    out = []
    for r in range(world):
        lo = min(bounds[r] * TILE, n_docs)
        hi = min(bounds[r + 1] * TILE, n_docs)
        out.append((lo, hi))
    return out


def pairs_in_rows(n_docs: int, lo: int, hi: int) -> int:
    """Number of i<j pairs with lo <= i < hi."""
    if hi <= lo:
        return 0
    return (hi - lo) * (n_docs - 1) - (hi * (hi - 1) // 2 - lo * (lo - 1) // 2)


def gather_sorted_keys(local_keys, world: int, all_gather_object) -> "list":
    """Concatenate the ranks' sorted key arrays in rank order (the global sorted
    candidate list, since ranks own increasing row ranges)."""
    parts = [None] * world
    all_gather_object(parts, local_keys)
    import numpy as np
    return np.concatenate([np.asarray(p, dtype=np.uint64) for p in parts]) if parts else np.zeros(0, np.uint64)


# ---------------------------------------------------------------------------
# Sharded K1/K2: each rank counts and signs a contiguous shard
# of the documents; the exchange steps are one all-reduce of df[V] (before
# IDF) and one all-gather of the signatures (before the pair triangle). With
# NCCL both run on device buffers (NVLink); the reference documents (K small
# docs) are counted by every rank from their tokens. The result is
# bit-identical to the single-GPU step: idf from the same global df table,
# reference rows weighted by the same kernel, S concatenated in document order.

def doc_shards(doc_off, world: int) -> list[tuple[int, int]]:
    """Contiguous document ranges [lo, hi) with about equal token counts."""
    import numpy as np
    off = np.asarray(doc_off, np.int64)
    n = len(off) - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    total = int(off[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        i = int(np.searchsorted(off, target, side="left"))
        if i > 0 and (i > n or abs(off[i - 1] - target) <= abs(off[min(i, n)] - target)):
            i -= 1
        cuts.append(min(max(cuts[-1], i), n))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def shard_corpus(tokens, doc_off, lo: int, hi: int):
    """(tokens, doc_off) of documents [lo, hi), offsets rebased to 0."""
    import numpy as np
    off = np.asarray(doc_off, np.uint64)
    b, e = int(off[lo]), int(off[hi])
    return np.asarray(tokens)[b:e], (off[lo:hi + 1] - np.uint64(b)).astype(np.uint64)


def reference_rows(ref_ctx, tokens, doc_off, ref_ids, vocab: int):
    """(rowptr, ids, counts) of the K reference documents, counted on the GPU
    by a small context from their tokens (every rank does this itself)."""
    import numpy as np
    off = np.asarray(doc_off, np.uint64)
    parts = [np.asarray(tokens)[int(off[d]):int(off[d + 1])] for d in ref_ids]
    r_off = np.zeros(len(parts) + 1, np.uint64)
    r_off[1:] = np.cumsum([len(p) for p in parts])
    r_tok = np.concatenate(parts).astype(np.uint32) if parts else np.zeros(0, np.uint32)
    ref_ctx.load_corpus(r_tok, r_off, vocab)
    ref_ctx.count(0)  # raw counts; weighting happens in the shard context
    return ref_ctx.counts()


class LocalComm:
    """In-process stand-in for the collectives: all 'ranks' live in this
    process (tests and single-GPU emulation of the sharded path)."""

    def allreduce_df(self, ctxs):
        import numpy as np
        tot = np.zeros(ctxs[0].vocab, np.uint64)
        for c in ctxs:
            tot += c.df()[0]
        return tot.astype(np.uint32)

    def allgather_signatures(self, ctxs):
        import numpy as np
        return np.concatenate([c.signatures() for c in ctxs], axis=0)


class _DevView:
    """__cuda_array_interface__ over a library device buffer (zero copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class TorchComm:
    """torch.distributed collectives. With the NCCL backend the df table and
    the signatures are reduced / gathered in place on the device (the
    library's buffers viewed as torch tensors through __cuda_array_interface__);
    with gloo they go through host arrays."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.nccl = dist.get_backend() == "nccl"
        self.device = device

    def allreduce_df(self, ctx):
        """Sum the shards' df tables; returns None when reduced in place on the
        device, else the global table (host) for set_global_df."""
        import numpy as np
        import torch
        import paper_1810_03099_b200 as R
        if self.nccl:
            ptr, nbytes = ctx.device_buffer(R.BUF_DF)
            t = torch.as_tensor(_DevView(ptr, (nbytes // 4,), "<i4"), device=self.device)
            ctx.synchronize()
            self.dist.all_reduce(t)
            torch.cuda.current_stream(self.device).synchronize()
            return None
        d = torch.from_numpy(ctx.df()[0].astype(np.int64))
        self.dist.all_reduce(d)
        return d.numpy().astype(np.uint32)

    def allgather_signatures(self, ctx, n_local: int, K: int, n_max: int):
        """Rank-ordered S of all shards: a device tensor [world*n_max, K] (NCCL)
        or a host array; returns (buffer, per-rank counts)."""
        import numpy as np
        import torch
        import paper_1810_03099_b200 as R
        world = self.dist.get_world_size()
        counts = [None] * world
        self.dist.all_gather_object(counts, n_local)
        if self.nccl:
            ptr, nbytes = ctx.device_buffer(R.BUF_SIGNATURES)
            mine = torch.zeros((n_max, K), dtype=torch.float32, device=self.device)
            if n_local:
                mine[:n_local] = torch.as_tensor(_DevView(ptr, (n_local, K), "<f4"), device=self.device)
            out = torch.empty((world * n_max, K), dtype=torch.float32, device=self.device)
            ctx.synchronize()
            self.dist.all_gather_into_tensor(out, mine)
            rows = torch.cat([out[r * n_max:r * n_max + counts[r]] for r in range(world)])
            return rows.contiguous(), counts
        S = np.zeros((n_max, K), np.float32)
        if n_local:
            S[:n_local] = ctx.signatures()
        parts = [None] * world
        self.dist.all_gather_object(parts, S)
        return np.concatenate([parts[r][:counts[r]] for r in range(world)]), counts


def sharded_signatures(shard_ctx, ref_ctx, tokens, doc_off, vocab: int, ref_ids, lo: int, hi: int,
                       n_global: int, weighting: int, global_df_fn):
    """Count + IDF(global df) + reference + sign for documents [lo, hi) of the
    corpus; `global_df_fn(shard_ctx)` performs the df exchange (returns the
    global table, or None when it was reduced in place)."""
    t, o = shard_corpus(tokens, doc_off, lo, hi)
    shard_ctx.load_corpus(t, o, vocab)
    shard_ctx.count(weighting)
    shard_ctx.set_global_df(n_global, global_df_fn(shard_ctx))
    rp, ids, cnt = reference_rows(ref_ctx, tokens, doc_off, ref_ids, vocab)
    shard_ctx.set_reference_counts(rp, ids, cnt)
    shard_ctx.sign(fetch=False)
