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


MIRRORS = {"PfConfig": "pf_config", "PfVertices": "pf_vertices", "PfTable": "pf_table",
           "PfKeyOut": "pf_key_out", "PfFrameBuffers": "pf_frame_buffers",
           "PfShard": "pf_shard", "PfReplica": "pf_replica", "PfScene": "pf_scene",
           "PfTraceOptions": "pf_trace_options", "PfPathOut": "pf_path_out",
           "PfEvictEvent": "pf_evict_event"}


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """Every ctypes mirror in _lib.py has the C compiler's sizeof and offsetof for
    every field of the header's struct (a probe compiled with gcc against
    include/pathfilter_b200.h), so header/ctypes drift fails here."""
    from paper_1902_05942_b200 import _lib
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "pathfilter_b200.h"',
             "int main(void) {"]
    want = {}
    for py, c in MIRRORS.items():
        cls = getattr(_lib, py)
        lines.append(f'printf("{c} sizeof %zu\\n", sizeof({c}));')
        want[(c, "sizeof")] = ctypes.sizeof(cls)
        for name, _ in cls._fields_:
            lines.append(f'printf("{c} {name} %zu\\n", offsetof({c}, {name}));')
            want[(c, name)] = getattr(cls, name).offset
    lines += ["return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                             check=True).stdout.splitlines():
        c, name, v = ln.split()
        got[(c, name)] = int(v)
    bad = {k: (got.get(k), v) for k, v in want.items() if got.get(k) != v}
    assert not bad, f"(C, ctypes) mismatches: {bad}"


@pytest.mark.parametrize("fs,sp,bv", [(0.003, 8.0, 0.02), (0.01, 8.0, 0.01), (1e-7, 3.0, 0.5),
                                      (0.0, 8.0, 0.01), (1e300, 8.0, 1e-10),
                                      (1e-310, 1.0, 1.0)])
def test_prepare_config_lod_dist(fs, sp, bv):
    """pf_prepare_config's lod_dist[k] is the smallest distance whose RN(d * c_lod)
    reaches the LOD threshold T[k] -- the bound make_key uses to skip the exact LOD of
    the jittered distance (checked in Python's own IEEE doubles)."""
    import math
    from paper_1902_05942_b200 import _lib
    from paper_1902_05942_b200.keys import FilterConfig
    cfg = FilterConfig(footprint_scale=fs, s_pixels=sp, base_voxel=bv)
    cin = cfg.to_c()
    out = _lib.PfConfig()
    L = _lib.lib()
    assert L.pf_prepare_config(ctypes.byref(cin), ctypes.byref(out)) == 0
    c = cin.c_lod
    assert out.inv_base_voxel == 1.0 / bv
    for k in range(0, 32):
        t = math.inf if k == 0 else cin.lod_threshold[k]  # [0]: where the ratio overflows
        d = out.lod_dist[k]
        if not 0.0 < c < math.inf:
            assert math.isnan(d)
        elif math.isinf(d):
            assert not (1.7976931348623157e308 * c >= t)
        else:
            assert d * c >= t
            assert d == 0.0 or math.nextafter(d, 0.0) * c < t
