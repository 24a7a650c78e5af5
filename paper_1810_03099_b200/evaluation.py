"""Evaluation harness pieces around the GPU path (SPEC.md eval module, SURVEY
§8f row 3): the EvalReport fields, the CSV of SPEC.md:444, and candidate-set
precision / recall against the exact-cosine ground truth.

The all-pairs error statistics themselves (MAE, mean error, variance: Eq. 2/3)
are fused on the GPU by Context.evaluate (refsig_gpu_evaluate); this module
only formats and compares.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass, fields

import numpy as np

CSV_HEADER = ["method", "partitions", "ngrams", "mae", "variance", "mean_error", "pairs", "avg_compare_us",
              "sign_ms", "sig_bytes"]


@dataclass
class EvalReport:
    """SPEC.md EvalReport: invariants variance >= 0 and mae >= |mean_error|."""
    method: str
    partitions: int  # K reference vectors (MRC) or 64 (Simhash bits)
    ngrams: int      # reference size in terms (union U) or 0
    mae: float
    variance: float
    mean_error: float
    pairs: int
    avg_compare_us: float
    sign_ms: float
    sig_bytes: int

    def check(self) -> None:
        if self.variance < 0 or self.mae + 1e-12 < abs(self.mean_error):
            raise ValueError(f"EvalReport invariants violated: {self}")


def reports_from_gpu(ev: dict, *, K: int, union: int, compare_s: float, sign_ms: float, n_docs: int,
                     fp_ms: float = 0.0) -> list[EvalReport]:
    """EvalReports for MRC and (if present) Simhash from Context.evaluate's
    dict. compare_s: device seconds of one all-pairs compare pass."""
    pairs = int(ev["pairs"])
    out = [EvalReport("mrc", K, union, ev["mrc_mae"], ev["mrc_variance"], ev["mrc_mean_error"], pairs,
                      1e6 * compare_s / max(pairs, 1), sign_ms, 8 * K * n_docs)]
    if not np.isnan(ev.get("simhash_mae", float("nan"))):
        out.append(EvalReport("simhash", 64, 0, ev["simhash_mae"], ev["simhash_variance"], ev["simhash_mean_error"],
                              pairs, 1e6 * compare_s / max(pairs, 1), fp_ms, 8 * n_docs))
    for r in out:
        r.check()
    return out


def report_csv(reports: list[EvalReport], path: str) -> None:
    """SPEC.md report_csv: header + one line per report."""
    if not reports:
        raise ValueError("report_csv needs at least one report")
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(CSV_HEADER)
        for r in reports:
            w.writerow([getattr(r, k) if not isinstance(getattr(r, k), float) else repr(getattr(r, k))
                        for k in CSV_HEADER])


def read_csv(path: str) -> list[EvalReport]:
    """Parse a report_csv file back (the SPEC's round-trip property)."""
    types = {f.name: f.type for f in fields(EvalReport)}
    out = []
    with open(path, newline="") as f:
        rd = csv.DictReader(f)
        if rd.fieldnames != CSV_HEADER:
            raise ValueError(f"unexpected header {rd.fieldnames}")
        for row in rd:
            vals = {}
            for k, v in row.items():
                t = types[k]
                vals[k] = v if t in ("str", str) else (int(v) if t in ("int", int) else float(v))
            out.append(EvalReport(**vals))
    return out


def precision_recall(candidates: np.ndarray, truth: np.ndarray) -> dict:
    """Candidate pair keys (sorted (i<<32)|j) against the ground-truth keys
    (e.g. exact cosine >= tau_cos): precision, recall, counts."""
    c = np.asarray(candidates, np.uint64)
    t = np.asarray(truth, np.uint64)
    tp = int(np.intersect1d(c, t, assume_unique=True).size)
    return {"candidates": int(c.size), "truth": int(t.size), "true_positives": tp,
            "precision": tp / c.size if c.size else float("nan"),
            "recall": tp / t.size if t.size else float("nan")}
