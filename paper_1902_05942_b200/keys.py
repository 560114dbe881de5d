"""Filter keys on the device: LOD, tangent-plane jitter, quantisation, hashing.

Mirrors the reference module src/keys.py (same names, argument meaning and
errors).  Every array result is a CUDA tensor computed by the sm_100a key kernel
(csrc/pf_table.cu: keys_kernel / hash_kernel); `KeyArrays.numpy()` gives the
reference dtypes (uint64 index, uint32 fingerprint).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib

SENTINEL = 0
MAX_LEVEL = 31

# T[k] = smallest double r with floor(np.log2(r)) >= k (numpy 2.3 in this image; numpy's
# log2 rounds up to k for a few doubles just below 2^k, so floor(log2) is not the
# exponent there).  Found by bisection over doubles; re-derived in tests/test_keys_cpu.py.
LOD_THRESHOLDS = tuple(float.fromhex(h) for h in (
    "0x1.0000000000000p+1", "0x1.0000000000000p+2", "0x1.fffffffffffffp+2",
    "0x1.fffffffffffffp+3", "0x1.ffffffffffffep+4", "0x1.ffffffffffffep+5",
    "0x1.ffffffffffffep+6", "0x1.ffffffffffffep+7", "0x1.ffffffffffffbp+8",
    "0x1.ffffffffffffbp+9", "0x1.ffffffffffffbp+10", "0x1.ffffffffffffbp+11",
    "0x1.ffffffffffffbp+12", "0x1.ffffffffffffbp+13", "0x1.ffffffffffffbp+14",
    "0x1.ffffffffffffbp+15", "0x1.ffffffffffff5p+16", "0x1.ffffffffffff5p+17",
    "0x1.ffffffffffff5p+18", "0x1.ffffffffffff5p+19", "0x1.ffffffffffff5p+20",
    "0x1.ffffffffffff5p+21", "0x1.ffffffffffff5p+22", "0x1.ffffffffffff5p+23",
    "0x1.ffffffffffff5p+24", "0x1.ffffffffffff5p+25", "0x1.ffffffffffff5p+26",
    "0x1.ffffffffffff5p+27", "0x1.ffffffffffff5p+28", "0x1.ffffffffffff5p+29",
    "0x1.ffffffffffff5p+30"))

_TEMPORAL = {"integrate": 0, "filter": 1, "hybrid": 2}


@dataclass
class FilterConfig:
    """Everything the key/table/pipeline stages agree on (src/keys.py:30-79)."""

    s_pixels: float = 8.0
    include_normal: bool = True
    normal_bins: int = 8
    include_incident_angle: bool = False
    incident_angle_bins: int = 4
    include_layer: bool = False
    normal_in_fingerprint: bool = False
    jitter: bool = True
    base_voxel: float = 0.01
    footprint_scale: float = 0.01
    capacity: int = 1 << 13
    probe_limit: int = 32
    low_count_threshold: int = 8
    temporal_mode: str = "integrate"
    ema_alpha: float = 0.8
    sum_mode: str = "fixed"
    multi_level: bool = True
    coarse_delta: int = 2
    evict_horizon: int = 8
    evict_min_age: int = 3
    delta_max: float = 0.5
    delta_eps: float = 1e-4
    alpha_refine: float = 0.25
    reevaluate_fraction: float = 1.0 / 16.0
    sample_cap: int = 256

    def __post_init__(self):
        if self.capacity < 1 or self.capacity & (self.capacity - 1):
            raise ValueError("capacity must be a power of two")
        if self.probe_limit < 1:
            raise ValueError("probe_limit must be >= 1")
        if self.s_pixels <= 0:
            raise ValueError("s_pixels must be positive")
        if self.temporal_mode not in _TEMPORAL:
            raise ValueError(f"unknown temporal_mode {self.temporal_mode!r}")
        if self.sum_mode not in ("fixed", "float"):
            raise ValueError(f"unknown sum_mode {self.sum_mode!r}")
        if not 0.0 <= self.ema_alpha <= 1.0:
            raise ValueError("ema_alpha must be in [0, 1]")

    def for_camera(self, fov: float, image_height: int) -> "FilterConfig":
        """Copy with footprint_scale derived from a camera (src/keys.py:74-76)."""
        return replace(self, footprint_scale=2.0 * math.tan(fov / 2.0) / image_height)

    def voxel_size(self, level: int) -> float:
        return self.base_voxel * float(2 ** level)

    def to_c(self) -> _lib.PfConfig:
        """The pf_config the kernels read; c_lod evaluated as src/keys.py:246 does.
        Cached per field values (it is rebuilt only when a knob changes)."""
        key = tuple(getattr(self, f) for f in self.__dataclass_fields__)
        cached = self.__dict__.get("_c_cache")
        if cached is not None and cached[0] == key:
            return cached[1]
        c = self._build_c()
        self.__dict__["_c_cache"] = (key, c)
        return c

    def _build_c(self) -> _lib.PfConfig:
        c = _lib.PfConfig()
        c.c_lod = self.footprint_scale * self.s_pixels / self.base_voxel
        c.base_voxel = float(self.base_voxel)
        c.ema_alpha = float(self.ema_alpha)
        c.delta_max = float(self.delta_max)
        c.lod_threshold[0] = 1.0
        for k, t in enumerate(LOD_THRESHOLDS, start=1):
            c.lod_threshold[k] = t
        c.normal_bins = int(self.normal_bins)
        c.incident_angle_bins = int(self.incident_angle_bins)
        c.include_normal = int(bool(self.include_normal))
        c.include_incident_angle = int(bool(self.include_incident_angle))
        c.include_layer = int(bool(self.include_layer))
        c.normal_in_fingerprint = int(bool(self.normal_in_fingerprint))
        c.jitter = int(bool(self.jitter))
        c.multi_level = int(bool(self.multi_level))
        c.coarse_delta = int(self.coarse_delta)
        c.low_count_threshold = int(self.low_count_threshold)
        c.temporal_mode = _TEMPORAL[self.temporal_mode]
        c.sample_cap = int(self.sample_cap)
        return c


def temporal_code(mode: str) -> int:
    if mode not in _TEMPORAL:
        raise ValueError(f"unknown temporal mode {mode!r}")
    return _TEMPORAL[mode]


@dataclass(frozen=True)
class CellKey:
    qx: int
    qy: int
    qz: int
    level: int
    aux: int = 0

    def neighbor(self, dx: int, dy: int, dz: int) -> "CellKey":
        return CellKey(self.qx + dx, self.qy + dy, self.qz + dz, self.level, self.aux)


@dataclass(frozen=True)
class CellHashes:
    index: int
    fingerprint: int


def pack_aux(normal_bin: int = 0, angle_bin: int = 0, layer: int = 0) -> int:
    return normal_bin | (angle_bin << 16) | (layer << 24)


# ------------------------------------------------------------------ tensor helpers

def device() -> torch.device:
    return _lib.require_cuda()


def as_f64(a, cols: int | None = None) -> torch.Tensor:
    """float64 contiguous CUDA tensor from numpy / torch input."""
    dev = device()
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, np.float64))
    t = t.to(device=dev, dtype=torch.float64).contiguous()
    if cols is not None and (t.dim() != 2 or t.shape[1] != cols):
        t = t.reshape(-1, cols)
    return t


def as_i64(a) -> torch.Tensor:
    """int64 contiguous CUDA tensor (uint64 numpy input keeps its bits)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.int64).contiguous()
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(dev)


def as_u32_bits(a) -> torch.Tensor:
    """uint32 fingerprints stored bit-for-bit in an int32 CUDA tensor."""
    dev = device()
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.int32:
            return a.to(dev).contiguous()
        return (a.to(device=dev, dtype=torch.int64) & 0xFFFFFFFF).to(torch.int32).contiguous()
    a = np.ascontiguousarray(a).astype(np.uint32, copy=False)
    return torch.from_numpy(a.view(np.int32).copy()).to(dev)


def u64_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def u32_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


@dataclass
class KeyArrays:
    """Struct-of-arrays CellKeys plus hashes (src/keys.py:302-320), on the device.

    index holds uint64 bits in an int64 tensor and fingerprint uint32 bits in an
    int32 tensor; numpy() returns the reference dtypes."""

    qx: torch.Tensor
    qy: torch.Tensor
    qz: torch.Tensor
    level: torch.Tensor
    aux: torch.Tensor
    index: torch.Tensor
    fingerprint: torch.Tensor
    jittered: torch.Tensor

    def __len__(self):
        return int(self.qx.shape[0])

    def cell_key(self, i: int) -> CellKey:
        return CellKey(int(self.qx[i]), int(self.qy[i]), int(self.qz[i]), int(self.level[i]),
                       int(self.aux[i]) & 0xFFFFFFFFFFFFFFFF)

    def numpy(self) -> dict:
        return {"qx": self.qx.cpu().numpy(), "qy": self.qy.cpu().numpy(),
                "qz": self.qz.cpu().numpy(), "level": self.level.cpu().numpy(),
                "aux": u64_numpy(self.aux), "index": u64_numpy(self.index),
                "fingerprint": u32_numpy(self.fingerprint),
                "jittered": self.jittered.cpu().numpy()}


def _empty_keys(n: int) -> KeyArrays:
    dev = device()
    e = lambda dt: torch.empty(n, dtype=dt, device=dev)  # noqa: E731
    return KeyArrays(e(torch.int64), e(torch.int64), e(torch.int64), e(torch.int64),
                     e(torch.int64), e(torch.int64), e(torch.int32),
                     torch.empty((n, 3), dtype=torch.float64, device=dev))


def _key_out(k: KeyArrays) -> _lib.PfKeyOut:
    o = _lib.PfKeyOut()
    for f in ("qx", "qy", "qz", "level", "aux", "index", "fingerprint", "jittered"):
        setattr(o, f, getattr(k, f).data_ptr())
    return o


def vertices_c(position, normal, omega_r, layer_id, camera_distance, pixel=None, sample=None,
               contribution=None, throughput=None) -> tuple[_lib.PfVertices, list]:
    """pf_vertices over CUDA tensors; returns the struct and the tensors it borrows."""
    keep = [position, normal, omega_r, layer_id, camera_distance, pixel, sample, contribution,
            throughput]
    v = _lib.PfVertices()
    v.position = _lib.ptr(position)
    v.normal = _lib.ptr(normal)
    v.omega_r = _lib.ptr(omega_r)
    v.contribution = _lib.ptr(contribution)
    v.throughput = _lib.ptr(throughput)
    v.pixel = _lib.ptr(pixel)
    v.sample = _lib.ptr(sample)
    v.layer_id = _lib.ptr(layer_id)
    v.camera_distance = _lib.ptr(camera_distance)
    v.n = int(camera_distance.shape[0])
    return v, keep


def make_key_arrays(position, normal, omega_r, layer_id, camera_distance,
                    cfg: FilterConfig, u1=None, u2=None, level_delta: int = 0) -> KeyArrays:
    """Vectorised make_cell_key + hashes over a vertex stream (src/keys.py:342-359)."""
    pos = as_f64(position, 3)
    nrm = as_f64(normal, 3)
    om = as_f64(omega_r, 3)
    lay = as_i64(layer_id)
    dist = as_f64(camera_distance).reshape(-1)
    n = int(dist.shape[0])
    zeros = torch.zeros(n, dtype=torch.int64, device=pos.device)
    v, keep = vertices_c(pos, nrm, om, lay, dist, pixel=zeros, sample=zeros)
    out = _empty_keys(n)
    d1 = as_f64(u1).reshape(-1) if (cfg.jitter and u1 is not None) else None
    d2 = as_f64(u2).reshape(-1) if (cfg.jitter and u1 is not None) else None
    ko = _key_out(out)
    _lib.call("pf_make_key_arrays", ctypes.byref(cfg.to_c()), ctypes.byref(v), _lib.ptr(d1),
              _lib.ptr(d2), int(level_delta), ctypes.byref(ko), _lib.stream_handle())
    del keep
    return out


# ------------------------------------------------------------------ vectorised stages
# The reference's per-stage numpy helpers (src/keys.py:245-300).  levels / bins / aux come
# from the key kernel itself (the fields it computes on the way to the hash), so they are
# the exact values the filter uses; jittered_positions restates the numpy expression as
# one device op per numpy op (no contraction across ops) with glibc-exact sin/cos.

def _stage_keys(n_or_dist, cfg: FilterConfig, normal=None, omega_r=None, layer_id=None
                ) -> KeyArrays:
    dist = as_f64(n_or_dist).reshape(-1)
    n = int(dist.shape[0])
    z3 = torch.zeros((n, 3), dtype=torch.float64, device=dist.device)
    nrm = as_f64(normal, 3) if normal is not None else z3
    om = as_f64(omega_r, 3) if omega_r is not None else z3
    lay = as_i64(layer_id).reshape(-1) if layer_id is not None else \
        torch.zeros(n, dtype=torch.int64, device=dist.device)
    return make_key_arrays(z3, nrm, om, lay, dist, replace(cfg, jitter=False))


def levels_array(camera_distance, cfg: FilterConfig) -> torch.Tensor:
    """LOD level per vertex, min(floor(log2(max(d * c_lod, 1))), 31) (src/keys.py:245-248)."""
    return _stage_keys(camera_distance, cfg).level


def normal_bins_array(n, bins: int) -> torch.Tensor:
    """Octahedral normal bin per row (src/keys.py:273-284)."""
    nrm = as_f64(n, 3)
    if int(bins) < 1:
        raise ValueError("bins must be >= 1")
    cfg = FilterConfig(include_normal=True, normal_bins=int(bins), normal_in_fingerprint=False,
                       include_incident_angle=False, include_layer=False, jitter=False)
    return _stage_keys(torch.ones(nrm.shape[0], dtype=torch.float64, device=nrm.device), cfg,
                       normal=nrm).aux


def aux_bits_array(normal, omega_r, layer_id, cfg: FilterConfig) -> torch.Tensor:
    """Packed aux field: normal bin | angle bin << 16 | layer << 24 (src/keys.py:286-300).
    int64 tensor holding the reference's uint64 values (all < 2^32)."""
    nrm = as_f64(normal, 3)
    return _stage_keys(torch.ones(nrm.shape[0], dtype=torch.float64, device=nrm.device), cfg,
                       normal=nrm, omega_r=omega_r, layer_id=layer_id).aux


def tangent_basis_array(n) -> tuple[torch.Tensor, torch.Tensor]:
    """Duff et al. orthonormal basis per row (src/keys.py:251-258)."""
    nrm = as_f64(n, 3)
    x, y, z = nrm[:, 0], nrm[:, 1], nrm[:, 2]
    s = torch.where(z >= 0.0, 1.0, -1.0).to(torch.float64)
    a = -1.0 / (s + z)
    b = (x * y) * a
    t1 = torch.stack([1.0 + ((s * x) * x) * a, s * b, -s * x], 1)
    t2 = torch.stack([b, s + (y * y) * a, -y], 1)
    return t1, t2


def sincos_array(x) -> tuple[torch.Tensor, torch.Tensor]:
    """glibc-exact (sin, cos) of a float64 array on the device (csrc pf_sincos)."""
    t = as_f64(x).reshape(-1)
    s = torch.empty_like(t)
    c = torch.empty_like(t)
    _lib.call("pf_sincos", _lib.ptr(t), int(t.shape[0]), _lib.ptr(s), _lib.ptr(c),
              _lib.stream_handle())
    return s, c


def jittered_positions(position, normal, level, u1, u2, cfg: FilterConfig) -> torch.Tensor:
    """Disc jitter of radius half a voxel in the tangent plane (src/keys.py:261-270)."""
    pos = as_f64(position, 3)
    if not cfg.jitter:
        return pos
    nrm = as_f64(normal, 3)
    lv = as_i64(level).reshape(-1)
    r = 0.5 * torch.sqrt(as_f64(u1).reshape(-1))
    phi = (2.0 * math.pi) * as_f64(u2).reshape(-1)
    sn, cs = sincos_array(phi)
    u = r * cs
    v = r * sn
    t1, t2 = tangent_basis_array(nrm)
    step = cfg.base_voxel * torch.ldexp(torch.ones_like(r), lv)
    off = u[:, None] * t1
    off = off + v[:, None] * t2
    return pos + off * step[:, None]


def hash_arrays(qx, qy, qz, level, aux, normal_fp_bins=None):
    """Index hash (uint64 bits, int64 tensor) and fingerprint (uint32 bits, int32 tensor)
    of key fields (src/keys.py:327-339)."""
    tx, ty, tz, tl, ta = (as_i64(a).reshape(-1) for a in (qx, qy, qz, level, aux))
    n = int(tx.shape[0])
    fb = as_u32_bits(normal_fp_bins).reshape(-1) if normal_fp_bins is not None else None
    index = torch.empty(n, dtype=torch.int64, device=tx.device)
    fp = torch.empty(n, dtype=torch.int32, device=tx.device)
    _lib.call("pf_hash_arrays", _lib.ptr(tx), _lib.ptr(ty), _lib.ptr(tz), _lib.ptr(tl),
              _lib.ptr(ta), _lib.ptr(fb), n, index.data_ptr(), fp.data_ptr(),
              _lib.stream_handle())
    return index, fp


def hashes(key: CellKey, normal_fp_bin: int | None = None) -> CellHashes:
    """Index hash and fingerprint of one key (src/keys.py:219-234), on the device."""
    fb = None if normal_fp_bin is None else np.array([normal_fp_bin & 0x3F], np.uint32)
    u = lambda x: np.array([x & 0xFFFFFFFFFFFFFFFF], np.uint64)  # noqa: E731
    idx, fp = hash_arrays(u(key.qx), u(key.qy), u(key.qz), u(key.level), u(key.aux), fb)
    return CellHashes(int(u64_numpy(idx)[0]), int(u32_numpy(fp)[0]))
