"""The reference's one-vertex key helpers (src/keys.py:100-240), for API parity.

Plain Python on one vertex at a time, exactly as the reference's scalar path: callers
use them to inspect a single key, never on the frame path (which is the sm_100a key
kernel).  Note the scalar LOD computes ((d * footprint) * s_pixels) / base_voxel with
math.log2, so near LOD edges it can differ from the vectorised recipe -- as in the
reference.
"""

from __future__ import annotations

import math

import numpy as np

from .keys import MAX_LEVEL, SENTINEL, CellKey, FilterConfig, pack_aux


def level_of_detail(camera_distance: float, cfg: FilterConfig) -> int:
    """Voxel level whose size covers ~s_pixels projected pixels, clamped to [0, 31]."""
    if camera_distance <= 0.0:
        raise ValueError("camera_distance must be positive")
    ratio = camera_distance * cfg.footprint_scale * cfg.s_pixels / cfg.base_voxel
    return 0 if ratio <= 1.0 else min(int(math.floor(math.log2(ratio))), MAX_LEVEL)


def tangent_basis(n):
    """Branchless orthonormal frame around n (Duff et al.)."""
    x, y, z = (float(c) for c in n[:3])
    s = 1.0 if z >= 0.0 else -1.0
    a = -1.0 / (s + z)
    b = x * y * a
    return (np.array([1.0 + s * x * x * a, s * b, -s * x]), np.array([b, s + y * y * a, -y]))


def disc_offsets(u1, u2):
    """Two uniforms -> a point of the disc of radius 1/2."""
    r = 0.5 * np.sqrt(u1)
    phi = 2.0 * math.pi * u2
    return r * np.cos(phi), r * np.sin(phi)


def jitter_position(x, n, level: int, draws, cfg: FilterConfig):
    """x moved inside the tangent-plane disc of half a level-`level` voxel."""
    x = np.asarray(x, float)
    if not cfg.jitter:
        return x
    u, v = disc_offsets(float(draws[0]), float(draws[1]))
    t1, t2 = tangent_basis(n)
    return x + (u * t1 + v * t2) * cfg.voxel_size(level)


def normal_bin(n, bins: int) -> int:
    """Octahedral-map bin in [0, bins^2)."""
    x, y, z = (float(c) for c in n[:3])
    s = abs(x) + abs(y) + abs(z)
    if s == 0.0:
        return 0
    px, py, pz = x / s, y / s, z / s
    if pz < 0.0:
        px, py = ((1.0 - abs(py)) * (1.0 if px >= 0.0 else -1.0),
                  (1.0 - abs(px)) * (1.0 if py >= 0.0 else -1.0))
    return (min(int((py * 0.5 + 0.5) * bins), bins - 1) * bins
            + min(int((px * 0.5 + 0.5) * bins), bins - 1))


def incident_angle_bin(n, omega_r, bins: int) -> int:
    c = min(max(float(np.dot(np.asarray(n, float), np.asarray(omega_r, float))), 0.0), 1.0)
    return min(int(c * bins), bins - 1)


def aux_bits(v, cfg: FilterConfig) -> int:
    """Normal / incident-angle / layer bits of a vertex descriptor."""
    nb = (normal_bin(v.normal, cfg.normal_bins)
          if cfg.include_normal and not cfg.normal_in_fingerprint else 0)
    ab = (incident_angle_bin(v.normal, v.omega_r, cfg.incident_angle_bins)
          if cfg.include_incident_angle and v.layer_id == 1 else 0)
    return pack_aux(nb, ab, v.layer_id if cfg.include_layer else 0)


def quantize(x, voxel: float):
    return tuple(int(math.floor(x[c] / voxel)) for c in range(3))


def make_cell_key(v, cfg: FilterConfig, jitter_draws=None, level_delta: int = 0) -> CellKey:
    """Key of one vertex: jitter at the original level, re-level at the moved point
    (path length grown by the offset), quantise."""
    lvl = min(level_of_detail(v.camera_distance, cfg) + level_delta, MAX_LEVEL)
    p = np.asarray(v.position, float)
    x = p
    if cfg.jitter and jitter_draws is not None:
        x = jitter_position(p, v.normal, lvl, jitter_draws, cfg)
        moved = v.camera_distance + float(np.linalg.norm(x - p))
        lvl = min(level_of_detail(moved, cfg) + level_delta, MAX_LEVEL)
    return CellKey(*quantize(x, cfg.voxel_size(lvl)), lvl, aux_bits(v, cfg))


def finalize_fingerprint(fp: int, normal_fp_bin: int | None = None) -> int:
    """Structured normal bits in the low six bits (optional) and the sentinel remap."""
    if normal_fp_bin is not None:
        fp = ((fp << 6) & 0xFFFFFFFF) | (normal_fp_bin & 0x3F)
    return SENTINEL + 1 if fp == SENTINEL else fp


def fingerprint_spatial_bits(fp: int) -> int:
    return fp >> 6
