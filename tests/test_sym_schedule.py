"""The symmetric sweep's visit protocol: ranks are a permutation per tile and
the list agents cannot deadlock (host model, tools/sym_schedule_check.py)."""
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
from sym_schedule_check import check  # noqa: E402


@pytest.mark.parametrize("n,sms", [(1100, 148), (20000, 148), (40000, 148), (100000, 148), (262144, 148),
                                   (5000, 8), (9999, 6), (30000, 10), (12345, 16), (70000, 132)])
def test_visit_protocol(n, sms):
    assert check(n, sms) == "ok"


@pytest.mark.parametrize("spread", [1, 4, 8])
def test_visit_protocol_spreads(spread):
    for n, sms in ((100000, 148), (30000, 10), (262144, 148)):
        assert check(n, sms, spread) == "ok"
