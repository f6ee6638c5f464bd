import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) shapes")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


# ---- parity error log: every GPU parity check records its worst normwise error here; with
# NB_PARITY_LOG=<path> the session writes them as JSON lines (test, case, kind, error)
_ERRS: list = []


def record(case, kind, err):
    if case is None:     # unnamed partial checks (e.g. one chunk of a full-size test) are not logged
        return
    test = os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
    _ERRS.append({"test": test, "case": case, "kind": kind, "err": float(err)})


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("NB_PARITY_LOG")
    if path and _ERRS:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            for e in _ERRS:
                f.write(json.dumps(e) + "\n")
