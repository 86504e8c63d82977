import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running case")


def pytest_collection_modifyitems(config, items):
    # A GPU test on a machine without CUDA is a hard skip only when the user
    # did not ask for -m gpu explicitly; with -m gpu a missing device fails.
    try:
        import torch

        have = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have = False
    markexpr = config.getoption("-m") or ""
    if have or "gpu" in markexpr.replace("not gpu", ""):
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(params=["restated", "reference"])
def oracle_backend(request):
    """Run an oracle test on the restatement (oracle/oracle.hpp) and on the
    reference's own hot-path code compiled in place (oracle/_ref, built by
    `make -C oracle ref` from /root/reference). The reference leg pins the
    restatement and the Python ports of the reference tests alike."""
    import oracle_py as O

    if request.param == "reference" and not O.reference_available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    with O.use_backend(request.param):
        yield request.param
