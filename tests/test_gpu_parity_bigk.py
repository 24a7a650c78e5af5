"""GPU parity of the compare rule (SPEC.md:369-377 over i<j) at
the K of configs[3] (K=64) and configs[4] (K=128), on BOTH K3 paths — the
tcgen05 split-fp16 kernel (k3_tc.cu) and the FP32 CUDA-core tiles
(k3_pairs.cu) — against the oracle (oracle/oracle.cpp orc_mrc_pairs /
orc_mrc_query_pairs, fp64).

Bar: candidate sets identical except pairs whose oracle score is within 1e-5
of tau, which the oracle lists (tests/parity_util.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
from tests.parity_util import BAND, assert_pairs_match

pytestmark = pytest.mark.gpu

PATHS = {"tensor": R.K3_TENSOR, "fp32": R.K3_FP32}


def _signed(ctx, cp, refs):
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    ctx.count()
    ctx.set_reference_docs(refs)
    return ctx.sign()


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("K", [42, 64, 100, 128])
def test_mrc_pairs_bigk_c0(gpu_ctx_factory, K, path):
    cp, cfg = C.config_corpus("c0")
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, K)
    ctx = gpu_ctx_factory()
    ctx.set_k3_path(PATHS[path])
    _signed(ctx, cp, refs)
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
    for tau in (0.9, 0.99):
        keys = ctx.mrc_pairs(tau)
        pairs, border = oracle.mrc_pairs(o.S, tau, BAND)
        assert_pairs_match(keys, pairs, border, f"c0 K={K} tau={tau} {path}")


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("K", [64, 128])
def test_mrc_pairs_bigk_c1_slice(gpu_ctx_factory, K, path):
    """5,000-document slice of configs[1] (20 topics, near-duplicates)."""
    cp, cfg = C.config_corpus("c1")
    cp = cp.slice_docs(5000)
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, K)
    ctx = gpu_ctx_factory()
    ctx.set_k3_path(PATHS[path])
    _signed(ctx, cp, refs)
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
    for tau in (0.9, 0.99):
        keys = ctx.mrc_pairs(tau)
        pairs, border = oracle.mrc_pairs(o.S, tau, BAND)
        assert_pairs_match(keys, pairs, border, f"c1[:5000] K={K} tau={tau} {path}")
    # a row panel (the streaming unit of configs[3]) equals the same rows of the full set
    k2 = ctx.mrc_pairs_rows(0.99, 1024, 2048)
    full = ctx.mrc_pairs(0.99)
    rows = full >> np.uint64(32)
    assert np.array_equal(k2, full[(rows >= 1024) & (rows < 2048)])


@pytest.mark.parametrize("path", list(PATHS))
def test_query_vs_database_k128(gpu_ctx_factory, path):
    """configs[4]'s K=128 query mode: queries x database rectangle (no triangle)."""
    cfg = C.load_configs()["configs"]["c4"]
    db_spec = dict(cfg["corpus"], n_docs=4000, vocab=50000)
    q_spec = dict(cfg["queries"], n_docs=600, vocab=50000)
    db = C.generate(db_spec)
    q = C.generate_queries(q_spec, db_spec, db)
    K = 128
    refs = C.sample_refs(0, db.n_docs, K)
    dbc = gpu_ctx_factory()
    Sd = _signed(dbc, db, refs)
    qc = gpu_ctx_factory()
    qc.set_k3_path(PATHS[path])
    qc.attach_database(dbc)
    qc.load_corpus(q.tokens, q.doc_off, q.vocab)
    qc.count()
    Sq = qc.sign()
    od = oracle.mrc_pipeline(db.tokens, db.doc_off, db.vocab, refs)
    xq = oracle.weighted(oracle.count(q.tokens, q.doc_off), od.idf)
    oSq = oracle.sign(xq, oracle.rows(od.x, refs))
    err = np.abs(Sq.astype(np.float64) - oSq)
    assert np.all(err <= 1e-5 * np.abs(oSq) + 1e-7)
    for tau in (0.9, 0.99):
        keys = qc.mrc_query_pairs(tau)
        pairs, border = oracle.mrc_query_pairs(oSq, od.S, tau, BAND)
        assert_pairs_match(keys, pairs, border, f"query K=128 tau={tau} {path}")


def test_mrc_pairs_c3_sampled_panel(gpu_ctx_factory):
    """configs[3] at full scale (200,000 docs, V=500k, K=64): signatures of
    every document within 1e-5, and the candidate set of rows [0, 2048) x all
    j > i (~4e8 pairs, ~48M candidates at tau=0.99) against the oracle."""
    cp, cfg = C.config_corpus("c3")
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    tau = C.load_configs()["thresholds"]["tau_mrc"]
    ctx = gpu_ctx_factory()
    S = _signed(ctx, cp, refs)
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
    err = np.abs(S.astype(np.float64) - o.S)
    assert np.all(err <= 1e-5 * np.abs(o.S) + 1e-7), f"max signature error {err.max():.3g}"
    keys = ctx.mrc_pairs_rows(tau, 0, 2048)
    pairs, border = oracle.mrc_pairs(o.S, tau, BAND, 0, 2048)
    nb = assert_pairs_match(keys, pairs, border, "c3 rows [0,2048)")
    print(f"c3 panel: {len(keys)} GPU pairs, {len(pairs)} oracle, {len(border)} in band, {nb} differ")


@pytest.mark.parametrize("K", [64, 128])
def test_evaluate_large_k_vs_oracle(gpu_ctx_factory, K):
    """SPEC eval with the MRC dot at K = 64 / 128 on tcgen05 (k5_tc.cu: head and
    MRC chains of one K walk) against the oracle's double-precision evaluation."""
    cp, cfg = C.config_corpus("c0")
    cp = cp.slice_docs(900)
    refs = C.sample_refs(1, cp.n_docs, K)
    ctx = gpu_ctx_factory()
    _signed(ctx, cp, refs)
    ctx.simhash(0)
    g = ctx.evaluate()
    o = oracle.mrc_pipeline(cp.tokens, cp.doc_off, cp.vocab, refs)
    fp = oracle.simhash(o.counts, o.idf, 0)
    ref = oracle.evaluate(o.x, o.S, fp)
    assert g["pairs"] == ref["pairs"]
    for k in ("mrc_mae", "mrc_mean_error", "simhash_mae", "simhash_mean_error"):
        assert abs(g[k] - ref[k]) <= 2e-6 + 1e-5 * abs(ref[k]), (k, g[k], ref[k])
    for k in ("mrc_variance", "simhash_variance"):
        assert abs(g[k] - ref[k]) <= 1e-7 + 1e-4 * abs(ref[k]), (k, g[k], ref[k])


_STRIPE_SNIPPET = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {repo!r})
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cfg = C.load_configs()["configs"]["c4"]
db_spec = dict(cfg["corpus"], n_docs=6000, vocab=50000)
q_spec = dict(cfg["queries"], n_docs={NQ}, vocab=50000)
db = C.generate(db_spec)
q = C.generate_queries(q_spec, db_spec, db)
refs = C.sample_refs(0, db.n_docs, {K})
with R.Context(0) as dbc, R.Context(0) as qc:
    dbc.load_corpus(db.tokens, db.doc_off, db.vocab); dbc.count(); dbc.set_reference_docs(refs); dbc.sign(fetch=False)
    qc.set_k3_path(R.K3_TENSOR)
    qc.attach_database(dbc)
    qc.load_corpus(q.tokens, q.doc_off, q.vocab); qc.count(); qc.sign(fetch=False)
    keys = qc.mrc_query_pairs(0.9)
print(len(keys), hashlib.sha256(np.ascontiguousarray(keys).tobytes()).hexdigest())
"""


@pytest.mark.parametrize("K,NQ", [(20, 700), (128, 700), (128, 600)])
def test_query_join_stripe_walk_equals_contiguous(K, NQ):
    """The stripe-major tile walk of the query rectangle (k3_tc.cu TileWalk,
    forced on with REFSIG_TC_STRIPE=1) gives the same candidate keys as the
    contiguous walk (REFSIG_TC_STRIPE=0), both paths of the tcgen05 kernel
    (K' <= 128 with two row blocks, chunked K' = 400), and so does the stripe
    walk in CTA pairs sharing every B chunk by cluster multicast
    (REFSIG_TC_MC=1, chunked path), and the cta_group::2 kernel (REFSIG_TC2=1:
    M = 256 over a CTA pair, each SM holding half of every B chunk; applies
    at K' > 128). 600 queries: an odd number of row blocks, so one CTA of a
    pair runs a ghost half."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _STRIPE_SNIPPET.format(repo=repo, K=K, NQ=NQ)
    out = {}
    for mode in ("0", "1", "mc", "pair"):
        env = dict(os.environ, REFSIG_TC_STRIPE="0" if mode == "0" else "1", REFSIG_TC_MC="1" if mode == "mc" else "0",
                   REFSIG_TC2="1" if mode == "pair" else "0")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = r.stdout.strip().splitlines()[-1]
    assert out["0"] == out["1"] == out["mc"] == out["pair"] and int(out["0"].split()[0]) > 0, out


_EMIT_SNIPPET = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {repo!r})
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
h = hashlib.sha256()
cp, cfg = C.config_corpus("c1")
cp = cp.slice_docs(6000)
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
with R.Context(0) as c:
    c.load_corpus(cp.tokens, cp.doc_off, cp.vocab); c.count(); c.set_reference_docs(refs); c.sign(fetch=False)
    for tau in (0.9, 0.99):
        k = c.mrc_pairs(tau); h.update(np.ascontiguousarray(k).tobytes()); print(len(k))
    c.simhash(0)
    k = c.hamming_pairs(12); h.update(np.ascontiguousarray(k).tobytes()); print(len(k))
print(h.hexdigest())
"""


def test_emit_wide_rows_equals_warp_per_row():
    """The CTA-per-row emitter for few wide rows (k3_pairs.cu emit_wide_kernel,
    forced with REFSIG_EMIT_WIDE=1) writes the same sorted candidates as the
    warp-per-row emitter (REFSIG_EMIT_WIDE=0): MRC at two thresholds (sparse
    and dense rows) and a Hamming join."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _EMIT_SNIPPET.format(repo=repo)
    out = {}
    for mode in ("0", "1"):
        env = dict(os.environ, REFSIG_EMIT_WIDE=mode)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = r.stdout.strip().splitlines()
    assert out["0"] == out["1"] and int(out["0"][0]) > 0, out


_PANEL_SNIPPET = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {repo!r})
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cp, cfg = C.config_corpus("c1")
cp = cp.slice_docs(5000)
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
with R.Context(0) as c:
    c.load_corpus(cp.tokens, cp.doc_off, cp.vocab); c.count(); c.set_reference_docs(refs); c.sign(fetch=False)
    c.simhash(0)
    k = c.exact_pairs(0.8)
    ev = c.evaluate()
print(len(k), hashlib.sha256(np.ascontiguousarray(k).tobytes()).hexdigest(), repr(ev["mrc_mae"]), repr(ev["simhash_variance"]))
"""


def test_exact_multi_panel_equals_single_panel():
    """K5's tail accumulator in several column panels (REFSIG_EXACT_PANEL=1024:
    five panels over 5,000 documents, the configs[3]-size path) gives the same
    exact pairs and the same evaluation sums as one panel (fixed-point tail
    sums: order-free, so bit-identical)."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _PANEL_SNIPPET.format(repo=repo)
    out = {}
    for panel in ("", "1024"):
        env = dict(os.environ)
        env.pop("REFSIG_EXACT_PANEL", None)
        if panel:
            env["REFSIG_EXACT_PANEL"] = panel
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[panel] = r.stdout.strip().splitlines()[-1]
    assert out[""] == out["1024"] and int(out[""].split()[0]) > 0, out


@pytest.mark.parametrize("name,n,K", [("c0", 0, 10), ("c1", 4000, 128)])
def test_self_join_pair_kernel_equals_single_cta(name, n, K):
    """The cta_group::2 kernel on the triangle (forced with REFSIG_TC2=1: the
    auto choice keeps it for the wide query join, where it is faster) writes
    the same candidates as the one-CTA tcgen05 kernel, at K' <= 128 and at
    K' = 400 (odd row-block counts run a ghost half)."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("0", "1"):
        env = dict(os.environ, REFSIG_TC2=mode)
        r = subprocess.run([sys.executable, os.path.join(repo, "tools", "tc2_self_probe.py"), name, str(n), str(K)],
                           env=env, capture_output=True, text=True, timeout=600, cwd=repo)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = r.stdout.strip().splitlines()
    assert out["0"] == out["1"] and int(out["0"][0]) > 0, out
