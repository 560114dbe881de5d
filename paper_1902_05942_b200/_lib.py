"""Loader for the sm_100a shared library `libpf_b200.so` (C ABI in include/pathfilter_b200.h).

There is no CPU fallback: importing a compute entry point without the built
library, or calling one without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("PF_LIB") or os.path.join(_PKG, "libpf_b200.so")
SOURCES = [os.path.join(_PKG, "csrc", f) for f in ("pf_common.cu", "pf_table.cu", "pf_frame.cu",
                                                    "pf_shard.cu", "pf_trace.cu")]
HEADERS = [os.path.join(_PKG, "csrc", f) for f in ("pf_device.cuh", "pf_insert.cuh",
                                                    "pf_sincos_tab.h",
                                                    "pf_internal.cuh", "pf_sweep.cuh",
                                                    "pf_resolve.cuh")] + \
    [os.path.join(_ROOT, "include", "pathfilter_b200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]

# exported symbols of include/pathfilter_b200.h (checked by tests/test_abi.py)
EXPORTS = ("pf_abi_version", "pf_last_error", "pf_device_sm_count", "pf_accumulate_fixed",
           "pf_accumulate_float", "pf_lookup_slots", "pf_make_key_arrays", "pf_vertex_keys",
           "pf_hash_arrays", "pf_insert_frame", "pf_resolve_frame", "pf_filter_frame",
           "pf_effective",
           "pf_begin_frame", "pf_check_contributions", "pf_selftest_division",
           "pf_count_occupied", "pf_finalize_image", "pf_shard_keys", "pf_shard_emit",
           "pf_shard_apply", "pf_shard_publish", "pf_replica_update", "pf_shard_reset",
           "pf_resolve_replica", "pf_trace_paths", "pf_sincos", "pf_segment_deltas",
           "pf_begin_frame_checked", "pf_prepare_config", "pf_build_id",
           "pf_host_register", "pf_host_unregister", "pf_accumulate_table",
           "pf_set_l2_persisting")

_BUILD_TAG = b"PF_BUILD_ID="


def source_id(extra_flags: tuple[str, ...] = ()) -> str:
    """SHA-256 (first 16 hex digits) of every source and header plus the nvcc flags:
    the identity a library built from this tree carries (pf_build_id)."""
    h = hashlib.sha256()
    for p in sorted(SOURCES + HEADERS):
        h.update(os.path.relpath(p, _ROOT).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS + list(extra_flags)).encode())
    return h.hexdigest()[:16]


def library_id(path: str = LIB_PATH) -> str | None:
    """The build id embedded in a built library (read from the file, not loaded)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        return None
    k = data.find(_BUILD_TAG)
    if k < 0:
        return None
    return data[k + len(_BUILD_TAG):k + len(_BUILD_TAG) + 16].decode(errors="replace")


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the CUDA sources for sm_100a into the in-tree shared library.  The
    library is rebuilt whenever its embedded build id differs from the tree's."""
    if not force and os.environ.get("PF_LIB") and os.path.exists(LIB_PATH):
        return LIB_PATH  # a prebuilt variant library (tools/build_variant.sh): never rebuilt
    sid = source_id()
    if not force and library_id() == sid:
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc, *NVCC_FLAGS, f"-DPF_BUILD_ID=\"{sid}\"", "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def build_id() -> str:
    """pf_build_id() of the loaded library."""
    return lib().pf_build_id().decode()


# ------------------------------------------------------------------ ctypes mirrors

class PfConfig(ctypes.Structure):
    _fields_ = [("c_lod", ctypes.c_double), ("base_voxel", ctypes.c_double),
                ("ema_alpha", ctypes.c_double), ("delta_max", ctypes.c_double),
                ("lod_threshold", ctypes.c_double * 32),
                ("normal_bins", ctypes.c_int32), ("incident_angle_bins", ctypes.c_int32),
                ("include_normal", ctypes.c_int32), ("include_incident_angle", ctypes.c_int32),
                ("include_layer", ctypes.c_int32), ("normal_in_fingerprint", ctypes.c_int32),
                ("jitter", ctypes.c_int32), ("multi_level", ctypes.c_int32),
                ("coarse_delta", ctypes.c_int32), ("low_count_threshold", ctypes.c_int32),
                ("temporal_mode", ctypes.c_int32), ("sample_cap", ctypes.c_int32),
                ("lod_ulps", ctypes.c_uint64 * 2), ("inv_base_voxel", ctypes.c_double),
                ("lod_dist", ctypes.c_double * 32)]


class PfVertices(ctypes.Structure):
    _fields_ = [("position", ctypes.c_void_p), ("normal", ctypes.c_void_p),
                ("omega_r", ctypes.c_void_p), ("contribution", ctypes.c_void_p),
                ("throughput", ctypes.c_void_p), ("pixel", ctypes.c_void_p),
                ("sample", ctypes.c_void_p), ("layer_id", ctypes.c_void_p),
                ("camera_distance", ctypes.c_void_p), ("n", ctypes.c_int64)]


class PfTable(ctypes.Structure):
    _fields_ = [("tags", ctypes.c_void_p), ("sums", ctypes.c_void_p),
                ("counts", ctypes.c_void_p), ("hist_sums", ctypes.c_void_p),
                ("hist_counts", ctypes.c_void_p), ("last_touch", ctypes.c_void_p),
                ("deltas", ctypes.c_void_p), ("capacity", ctypes.c_int64),
                ("sum_mode", ctypes.c_int32), ("probe_limit", ctypes.c_int32),
                ("evict_min_age", ctypes.c_int32), ("evict_horizon", ctypes.c_int32),
                ("cnt_stride", ctypes.c_int32), ("sum_stride", ctypes.c_int32),
                ("cold_stride", ctypes.c_int32), ("hsum_stride", ctypes.c_int32),
                ("sum_cstride", ctypes.c_int64)]


class PfKeyOut(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("qx", "qy", "qz", "level", "aux", "index",
                                                "fingerprint", "jittered")]


class PfFrameBuffers(ctypes.Structure):
    _fields_ = [("acc_stats", ctypes.c_void_p), ("res_stats", ctypes.c_void_p),
                ("events", ctypes.c_void_p), ("event_count", ctypes.c_void_p),
                ("event_capacity", ctypes.c_int64), ("bad_flag", ctypes.c_void_p),
                ("horizon_clears_fine", ctypes.c_void_p),
                ("horizon_clears_coarse", ctypes.c_void_p), ("lookup_keys", ctypes.c_void_p),
                ("eff_records", ctypes.c_void_p),
                ("flat", ctypes.c_void_p), ("work", ctypes.c_void_p),
                ("work_count", ctypes.c_void_p), ("fallback_keys", ctypes.c_void_p),
                ("phase_events", ctypes.c_void_p * 4),
                ("occ_in", ctypes.c_void_p * 2), ("occ_count_in", ctypes.c_void_p),
                ("occ_out", ctypes.c_void_p * 2), ("occ_count_out", ctypes.c_void_p)]


class PfShard(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("log2_capacity", ctypes.c_int32), ("sum_mode", ctypes.c_int32),
                ("agg_keys", ctypes.c_void_p), ("agg_sums", ctypes.c_void_p),
                ("agg_counts", ctypes.c_void_p), ("agg_capacity", ctypes.c_int64),
                ("distinct", ctypes.c_void_p), ("n_distinct", ctypes.c_void_p),
                ("overflow", ctypes.c_void_p), ("owner_counts", ctypes.c_void_p),
                ("owner_cursor", ctypes.c_void_p)]


class PfReplica(ctypes.Structure):
    _fields_ = [("fine_tags", ctypes.c_void_p), ("fine_records", ctypes.c_void_p),
                ("coarse_tags", ctypes.c_void_p), ("coarse_records", ctypes.c_void_p),
                ("capacity", ctypes.c_int64), ("slice_log2", ctypes.c_int32),
                ("probe_limit", ctypes.c_int32), ("sum_mode", ctypes.c_int32),
                ("pad0", ctypes.c_int32)]


class PfScene(ctypes.Structure):
    _fields_ = [("v0", ctypes.c_void_p), ("e1", ctypes.c_void_p), ("e2", ctypes.c_void_p),
                ("normal", ctypes.c_void_p), ("emission", ctypes.c_void_p),
                ("area", ctypes.c_void_p), ("material_id", ctypes.c_void_p),
                ("n_triangles", ctypes.c_int64), ("albedo", ctypes.c_void_p),
                ("glossy_weight", ctypes.c_void_p), ("glossy_exponent", ctypes.c_void_p),
                ("n_materials", ctypes.c_int64), ("light_tri", ctypes.c_void_p),
                ("n_lights", ctypes.c_int64), ("background", ctypes.c_double * 3),
                ("cam_pos", ctypes.c_double * 3), ("cam_right", ctypes.c_double * 3),
                ("cam_up", ctypes.c_double * 3), ("cam_fwd", ctypes.c_double * 3),
                ("ndc_scale_x", ctypes.c_double), ("ndc_scale_y", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class PfTraceOptions(ctypes.Structure):
    _fields_ = [("max_depth", ctypes.c_int32), ("rr_start", ctypes.c_int32),
                ("nee", ctypes.c_int32), ("select_k", ctypes.c_int32),
                ("pixel_jitter", ctypes.c_int32), ("pad0", ctypes.c_int32),
                ("rr_lo", ctypes.c_double), ("rr_hi", ctypes.c_double),
                ("diffuse_threshold", ctypes.c_double)]


class PfPathOut(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("radiance", ctypes.c_void_p),
                ("has_vertex", ctypes.c_void_p), ("position", ctypes.c_void_p),
                ("normal", ctypes.c_void_p), ("omega_r", ctypes.c_void_p),
                ("contribution", ctypes.c_void_p), ("throughput", ctypes.c_void_p),
                ("layer_id", ctypes.c_void_p), ("camera_distance", ctypes.c_void_p)]


class PfEvictEvent(ctypes.Structure):
    _fields_ = [("vertex", ctypes.c_int64), ("slot", ctypes.c_int64),
                ("victim_tag", ctypes.c_uint64), ("victim_touch", ctypes.c_int64)]


STAT_PROBE_FAILURES = 0
STAT_COARSE_PROBE_FAILURES = 1
STAT_PROBE_LEN_SUM = 2
STAT_EVICTIONS = 3
STAT_COARSE_EVICTIONS = 4
STAT_SOURCE_FINE = 5
STAT_SOURCE_NEIGHBORHOOD = 6
STAT_SOURCE_COARSE = 7
STAT_SOURCE_UNFILTERED = 8
STAT_FALLBACK_ROWS = 9
STAT_BAD_PIXELS = 10
STAT_SHARD_RECORDS = 11
STAT_SHARD_REQUESTS = 12
STAT_HIST_BASE = 16
WORK_LISTS = 64  # PF_WORK_LISTS


def work_rows(n: int) -> int:
    """PF_WORK_ROWS(n): entries of the resolve's work-list buffer for n vertices."""
    blocks = (int(n) + 255) // 256
    return max((blocks + WORK_LISTS - 1) // WORK_LISTS * WORK_LISTS * 256, 1)
STAT_COUNT = 16 + 256

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded library; raises if it is missing or no CUDA device is present."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    if not os.environ.get("PF_LIB"):
        want, have = source_id(), library_id()
        if have != want:
            raise RuntimeError(f"{LIB_PATH} was built from other sources (build id {have}, "
                               f"tree {want}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u64, dbl = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                              ctypes.c_uint64, ctypes.c_double)
    L.pf_abi_version.restype = ctypes.c_int
    L.pf_last_error.restype = ctypes.c_char_p
    L.pf_build_id.restype = ctypes.c_char_p
    L.pf_device_sm_count.restype = ctypes.c_int
    acc = [vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, i64, i64, i32, i32, i32,
           vp, vp, vp, vp, vp, vp]
    L.pf_accumulate_fixed.argtypes = acc
    L.pf_accumulate_float.argtypes = acc
    L.pf_lookup_slots.argtypes = [vp, i64, vp, vp, i64, i32, vp, vp]
    L.pf_accumulate_table.argtypes = [vp, vp, vp, vp, i64, i64, i32, vp, vp, vp, vp, vp, vp]
    L.pf_make_key_arrays.argtypes = [vp, vp, vp, vp, i32, vp, vp]
    L.pf_vertex_keys.argtypes = [vp, vp, u64, i32, vp, vp]
    L.pf_hash_arrays.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp, vp]
    L.pf_insert_frame.argtypes = [vp, vp, vp, vp, u64, i64, vp, vp, vp, i64, vp, u64, vp, vp]
    L.pf_resolve_frame.argtypes = [vp, vp, vp, vp, u64, u64, i64, vp, i64, vp, vp, vp, vp,
                                   vp, vp, vp, vp, vp, vp, vp]
    L.pf_filter_frame.argtypes = [vp, vp, vp, vp, i64, u64, u64, u64, i64, vp, i64, vp, vp, vp,
                                  vp, vp]
    L.pf_effective.argtypes = [vp, i32, dbl, dbl, vp, vp, vp]
    L.pf_begin_frame.argtypes = [vp, i64, i32, dbl, dbl, i32, vp, vp]
    L.pf_count_occupied.argtypes = [vp, i64, vp, vp]
    L.pf_check_contributions.argtypes = [vp, i64, vp, vp]
    L.pf_selftest_division.argtypes = [u64, i64, dbl, vp, vp]
    L.pf_finalize_image.argtypes = [vp, vp, vp, i64, i64, vp]
    L.pf_shard_keys.argtypes = [vp, vp, vp, i32, u64, u64, vp, vp, vp]
    L.pf_shard_emit.argtypes = [vp, vp, vp, vp]
    L.pf_shard_apply.argtypes = [vp, vp, vp, vp, i64, i64, vp, vp]
    L.pf_shard_publish.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.pf_replica_update.argtypes = [vp, vp, vp, i32, i64, i32, vp]
    L.pf_resolve_replica.argtypes = [vp, vp, vp, u64, u64, vp, vp, i64, i64, vp, vp, vp, vp,
                                     vp, vp, vp]
    L.pf_shard_reset.argtypes = [vp, vp]
    L.pf_trace_paths.argtypes = [vp, vp, u64, vp, vp, i64, vp, vp]
    L.pf_sincos.argtypes = [vp, i64, vp, vp, vp]
    L.pf_prepare_config.argtypes = [vp, vp]
    L.pf_host_register.argtypes = [vp, i64]
    L.pf_host_unregister.argtypes = [vp]
    L.pf_set_l2_persisting.argtypes = [i64, vp]
    L.pf_segment_deltas.argtypes = [vp, vp, i64, vp, vp, dbl, vp, vp]
    L.pf_begin_frame_checked.argtypes = [vp, vp, i64, i32, dbl, dbl, i32, vp, vp, vp, i64, vp,
                                         vp]
    for name in EXPORTS[3:]:
        if name != "pf_build_id":
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


_l2_done: dict = {}


def configure_l2() -> int:
    """Once per device: set aside L2 for evict_last lines (pf_set_l2_persisting).
    PF_L2_PERSIST_MB overrides the size (-1: the device maximum, 0: none)."""
    dev = torch.cuda.current_device()
    if dev in _l2_done:
        return _l2_done[dev]
    mb = int(os.environ.get("PF_L2_PERSIST_MB", "32"))
    got = ctypes.c_int64(0)
    call("pf_set_l2_persisting", mb if mb < 0 else mb << 20, ctypes.byref(got))
    _l2_done[dev] = got.value
    return got.value


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1902_05942_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


BACKEND = "b200"


def check_backend(name: str | None) -> None:
    """get_kernels (src/_backend.py:33-42): None or this build's name selects the device
    kernels; "native" (the reference's compiled backend) is accepted as an alias.  The
    reference's "python" backend is a CPU path and does not exist here."""
    if name is None or name in (BACKEND, "native"):
        return
    raise ValueError(f"unknown backend {name!r}")


def call(name: str, *args) -> None:
    """Invoke a C-ABI entry point and raise on a nonzero pf_status."""
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.pf_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle() -> int:
    """cudaStream_t of torch's current stream on the current device (the raw accessor:
    torch.cuda.current_stream() costs several microseconds per frame call)."""
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
