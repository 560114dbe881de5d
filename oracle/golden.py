"""ORACLE -- TEST INFRASTRUCTURE ONLY: loaders for the reference-generated fixtures
in tests/golden/ (shared by tests/ and __graft_entry__.smoke())."""

from __future__ import annotations

import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

STREAM_FIELDS = ("position", "normal", "omega_r", "contribution", "throughput", "pixel",
                 "sample", "layer_id", "camera_distance")
TABLE_FIELDS = ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas")


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
