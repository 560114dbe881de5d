"""C-ABI surface checks that need no GPU: the library builds for sm_100a, loads,
exports every entry point include/pathfilter_b200.h declares, and the ctypes
mirrors match the C struct layouts."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pathfilter_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1902_05942_b200 import _lib
    _lib.build()
    return ctypes.CDLL(_lib.LIB_PATH)


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(pf_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "pf_insert_frame" in names and "pf_accumulate_fixed" in names
    from paper_1902_05942_b200 import _lib
    assert sorted(_lib.EXPORTS) == names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(
        ROOT, "paper_1902_05942_b200", "libpf_b200.so")], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_abi_version_without_gpu(lib):
    lib.pf_abi_version.restype = ctypes.c_int
    import re
    with open(os.path.join(ROOT, "include", "pathfilter_b200.h")) as fh:
        want = int(re.search(r"#define PF_ABI_VERSION (\d+)", fh.read()).group(1))
    assert lib.pf_abi_version() == want


def test_argument_errors_are_status_codes(lib):
    """Invalid arguments return PF_ERR_ARGUMENT before touching the device."""
    lib.pf_lookup_slots.restype = ctypes.c_int
    lib.pf_last_error.restype = ctypes.c_char_p
    rc = lib.pf_lookup_slots(None, ctypes.c_int64(1000), None, None, ctypes.c_int64(4),
                             ctypes.c_int32(8), None, None)
    assert rc == 1
    assert b"power of two" in lib.pf_last_error()


def test_cubin_is_sm100a():
    so = os.path.join(ROOT, "paper_1902_05942_b200", "libpf_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    from paper_1902_05942_b200 import _lib
    assert ctypes.sizeof(_lib.PfConfig) == 4 * 8 + 32 * 8 + 12 * 4 + 2 * 8 + 8
    assert ctypes.sizeof(_lib.PfVertices) == 10 * 8
    assert ctypes.sizeof(_lib.PfTable) == 8 * 8 + 4 * 4
    assert ctypes.sizeof(_lib.PfEvictEvent) == 32
