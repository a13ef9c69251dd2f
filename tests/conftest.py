import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_worked_examples.json")) as f:
        return json.load(f)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Report every use of a conditioning floor (readings R4c / R6b): rows that passed the parity
    bar only with the floor, per check, and the totals."""
    try:
        from tests.parity import FLOOR_LOG
    except Exception:
        return
    if not FLOOR_LOG:
        return
    used = [(w, k, n) for w, k, n in FLOOR_LOG if k > 0]
    tot_k = sum(k for _, k, _ in FLOOR_LOG); tot_n = sum(n for _, _, n in FLOOR_LOG)
    terminalreporter.write_line(
        f"conditioning floors (R4c/R6b): {tot_k} of {tot_n} rows needed a floor, in {len(used)} of "
        f"{len(FLOOR_LOG)} floor-enabled checks")
    for w, k, n in used[:40]:
        terminalreporter.write_line(f"  floor used: {w}: {k}/{n} rows")
