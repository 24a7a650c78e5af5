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
