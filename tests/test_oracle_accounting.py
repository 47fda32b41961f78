"""Pins for oracle.accounting against values printed in the paper (tests/golden/*)."""
import os

import pytest

from oracle import para_saved, usage_ratio

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


PARA = _rows("para_saved_table_h.txt")
APPF = _rows("app_f_matched_memory.txt")


def test_fixture_sizes():
    assert len(PARA) == 52 and len(APPF) == 9


@pytest.mark.parametrize("row", PARA, ids=[r[0] for r in PARA])
def test_para_saved_table_h(row):
    """Table H "Para. Saved", both values, to the paper's two decimals."""
    _, n, method, r, clusters, per, total = row
    n = 10 if n == "-" else int(n)      # SVD rows do not depend on n
    p, t = para_saved(method, n, int(r), int(clusters))
    # printed to two decimals: the exact value must lie within half a unit of the last digit
    assert abs(p - float(per)) <= 0.005 + 1e-12
    assert abs(t - float(total)) <= 0.005 + 1e-12


@pytest.mark.parametrize("row", APPF, ids=[r[0] for r in APPF])
def test_app_f_matched_memory(row):
    """App F: usage ratio vs the matched vLLM max-gpu-lora."""
    _, n, method, r, clusters, slots = row
    ratio = usage_ratio(method, int(n), int(r), int(clusters))
    assert abs(ratio - int(slots)) < 1.0
    if int(n) in (32, 64):
        assert ratio == int(slots)          # exact anchors 5.0 and 6.0
