"""pytest plugin (test infrastructure): route the REFERENCE's kernel selection
(src/_backend.py:14-42) to this repo's sm_100a kernel module -- what INTEGRATION.md 1's
one-branch patch does -- so the reference's own tests run on the B200 kernels.

    python -m pytest -p dropin_plugin baseline/_ref/_ref_tests/test_table.py

Counts the calls that reached the device module and writes them to $PF_DROPIN_REPORT
at session end, so the caller can tell the tests really ran through it."""

import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)

import pathfilter  # noqa: E402
import pathfilter._backend as _backend  # noqa: E402

from paper_1902_05942_b200 import kernels as _b200  # noqa: E402

CALLS = {"accumulate_fixed": 0, "accumulate_float": 0, "lookup_slots": 0}


def _counted(name):
    fn = getattr(_b200, name)

    def wrapper(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)
    return wrapper


_module = types.SimpleNamespace(NAME=_b200.NAME, **{k: _counted(k) for k in CALLS},
                                intersect_closest=_b200.intersect_closest,
                                intersect_any=_b200.intersect_any)
_backend.kernels = _module
_backend.BACKEND = _module.NAME
pathfilter.BACKEND = _module.NAME


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PF_DROPIN_REPORT")
    if path:
        with open(path, "w") as fh:
            json.dump({"calls": CALLS, "backend": _backend.BACKEND}, fh)
