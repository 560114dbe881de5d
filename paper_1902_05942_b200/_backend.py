"""Backend selection (src/_backend.py:1-52).

The reference picks between a compiled extension ("native") and a numpy kernel
module ("python").  This build has one backend, the sm_100a kernels of libpf_b200.so;
"native" is accepted as its alias and anything else raises, as get_kernels does.
"""

from __future__ import annotations

from . import _lib
from ._lib import BACKEND


def available_backends() -> list:
    """The kernel backends this build provides (src/_backend.py:45-52)."""
    return [BACKEND]


def get_kernels(name: str | None = None):
    """The kernel library for `name` (src/_backend.py:33-42): the loaded libpf_b200.so."""
    _lib.check_backend(name)
    return _lib.lib()
