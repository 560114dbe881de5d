import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

STREAM_FIELDS = ("position", "normal", "omega_r", "contribution", "throughput", "pixel",
                 "sample", "layer_id", "camera_distance")
TABLE_FIELDS = ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C ABI)")


class Stream:
    """Plain numpy vertex stream with the reference VertexStream field names."""

    def __init__(self, **kw):
        for f in STREAM_FIELDS:
            setattr(self, f, kw[f])

    def __len__(self):
        return len(self.pixel)


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def golden_stream(d, prefix: str = "v_") -> Stream:
    return Stream(**{f: d[f"{prefix}{f}"] for f in STREAM_FIELDS})


def golden_cfg(d, key: str) -> dict:
    return json.loads(str(d[key]))


def golden_table(d, prefix: str) -> dict:
    return {f: d[f"{prefix}{f}"] for f in TABLE_FIELDS}


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
