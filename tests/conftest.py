import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # gpu tests are skipped (not failed) when no device is present, unless explicitly selected.
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Aggregate parity statistics of the GPU tests (tests/parity.py STATS): worst band /
    corr errors and the R3 near-tie accepts, shown even under -q."""
    mod = sys.modules.get("parity")
    if mod is None or not getattr(mod, "STATS", None):
        return
    st = mod.STATS
    tot = sum(s.get("lag_total", 0) for s in st)
    ex = sum(s.get("lag_exact", 0) for s in st)
    nt = sum(s.get("lag_neartie", 0) for s in st)
    terminalreporter.write_line(
        f"parity: {len(st)} comparisons, max band rel L2 {max(s['band_rel_l2'] for s in st):.2e}, "
        f"max corr err/peak {max(s['corr_err'] for s in st):.2e}, lags {ex}/{tot} exact, {nt} near-tie accepts")
