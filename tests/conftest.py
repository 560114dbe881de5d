import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.golden import GOLDEN, STREAM_FIELDS, TABLE_FIELDS, Stream, golden_cfg, \
    golden_stream, golden_table, load_golden  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C ABI)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pf_oracle
    pf_oracle.build_lib()
    return pf_oracle


@pytest.fixture(scope="session")
def gpu():
    """The product package on a CUDA device; fails loudly (never skips) without one."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1902_05942_b200 as pf
    return pf
