import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full BASELINE-size parity (minutes)")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "ref_kat.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def ref_fields():
    return dict(np.load(os.path.join(GOLDEN, "ref_fields.npz")))


@pytest.fixture(scope="session")
def big_digests():
    p = os.path.join(GOLDEN, "big_digests.json")
    if not os.path.exists(p):
        pytest.skip("big digests not generated")
    with open(p) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def O():
    from oracle import oracle
    oracle.build_c()
    return oracle


@pytest.fixture(scope="session")
def sp():
    import paper_0912_4506_b200 as sp
    sp._native.load_library()
    return sp
