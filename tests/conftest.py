import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def small_golden():
    with open(os.path.join(GOLDEN, "reference_small.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def full_golden():
    p = os.path.join(GOLDEN, "reference_full.json")
    if not os.path.exists(p):
        pytest.skip("reference_full.json not generated")
    with open(p) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def next_golden():
    """sparsification, per-edge counts, variance report."""
    with open(os.path.join(GOLDEN, "reference_next.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orders_golden():
    """Every OrderKind (order.hpp:17-128) through the reference."""
    with open(os.path.join(GOLDEN, "reference_orders.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def io_golden():
    """parse_edge_list / write_edge_list (io.hpp:18-64) through the reference."""
    with open(os.path.join(GOLDEN, "reference_io.json")) as f:
        return json.load(f)
