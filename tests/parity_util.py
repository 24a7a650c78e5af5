"""Shared parity helpers (test infrastructure; used by the gpu tests and
tools/border_pairs.py).

Candidate-set bar (north_star): the GPU set equals the oracle's
except for pairs whose oracle score lies within 1e-5 of the threshold; those
are listed by the oracle (`border`) and every disagreement must be one of
them. Sorted uint64 keys (i << 32 | j) are compared with numpy set algebra so
that panels of tens of millions of pairs stay cheap."""
import numpy as np

BAND = 1e-5


def _u64(a):
    return np.ascontiguousarray(a, np.uint64)


def pair_disagreements(gpu_keys, orc_keys):
    """(only_gpu, only_oracle) as sorted uint64 arrays."""
    g, o = _u64(gpu_keys), _u64(orc_keys)
    return np.setdiff1d(g, o, assume_unique=True), np.setdiff1d(o, g, assume_unique=True)


def assert_pairs_match(gpu_keys, orc_keys, border, label=""):
    """Returns the number of (allowed, listed) borderline disagreements."""
    g = _u64(gpu_keys)
    assert g.size < 2 or np.all(g[1:] > g[:-1]), f"{label}: GPU pairs not strictly sorted"
    only_g, only_o = pair_disagreements(g, orc_keys)
    diff = np.concatenate([only_g, only_o])
    outside = np.setdiff1d(diff, _u64(border))
    assert outside.size == 0, (f"{label}: {outside.size} pair mismatches outside the 1e-5 band "
                               f"(e.g. {[(int(k) >> 32, int(k) & 0xFFFFFFFF) for k in outside[:5]]})")
    return int(diff.size)


def border_listing(gpu_keys, orc_keys, border, S_rows, S_cols=None, tau=0.99, row_base=0):
    """Every pair the GPU and the oracle decide differently, with the oracle's
    score (fp64 compare of the oracle signatures) and both decisions."""
    import oracle
    only_g, only_o = pair_disagreements(gpu_keys, orc_keys)
    S_cols = S_rows if S_cols is None else S_cols
    out = []
    for keys, gpu_match in ((only_g, True), (only_o, False)):
        for k in keys.tolist():
            i, j = k >> 32, k & 0xFFFFFFFF
            score = float(oracle.compare(S_rows[i - row_base], S_cols[j]))
            out.append({"i": int(i), "j": int(j), "oracle_score": score, "score_minus_tau": score - tau,
                        "gpu_match": gpu_match, "oracle_match": not gpu_match})
    out.sort(key=lambda r: (r["i"], r["j"]))
    return out
