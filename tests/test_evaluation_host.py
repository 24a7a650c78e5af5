"""Host side of the evaluation harness (SPEC.md eval): CSV per SPEC.md:444
with the round-trip property, report invariants, precision/recall."""
import numpy as np
import pytest

from paper_1810_03099_b200 import evaluation as E


def test_csv_round_trip(tmp_path):
    reps = [E.EvalReport("mrc", 60, 1500, 0.12328, 0.01947, -0.01, 177197778, 0.004, 12.5, 480),
            E.EvalReport("simhash", 64, 0, 0.18854, 0.04173, 0.18, 177197778, 0.001, 3.0, 8)]
    p = tmp_path / "r.csv"
    E.report_csv(reps, str(p))
    lines = p.read_text().strip().splitlines()
    assert lines[0] == ",".join(E.CSV_HEADER) and len(lines) == 3  # SPEC: 2 reports -> 3-line CSV
    assert E.read_csv(str(p)) == reps
    with pytest.raises(ValueError):
        E.report_csv([], str(p))


def test_report_invariants():
    E.EvalReport("mrc", 1, 1, 0.1, 0.0, -0.1, 1, 0, 0, 8).check()
    with pytest.raises(ValueError):
        E.EvalReport("mrc", 1, 1, 0.05, 0.0, -0.1, 1, 0, 0, 8).check()  # mae < |mean_error|


def test_precision_recall():
    k = lambda i, j: (i << 32) | j
    cand = np.array([k(0, 1), k(0, 2), k(1, 2)], np.uint64)
    truth = np.array([k(0, 1), k(2, 3)], np.uint64)
    pr = E.precision_recall(cand, truth)
    assert pr["true_positives"] == 1 and pr["precision"] == pytest.approx(1 / 3) and pr["recall"] == 0.5
