"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference hashed path-space filter
(`/root/reference/pkg/src/pathfilter`, cited below as `src/<file>:<line>`).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module; the product package never does, and it must fail
loudly rather than fall back here.

Keys, effective sums, the temporal fold and the resolve ladder are numpy,
written op for op in the reference's evaluation order (so they share numpy's
libm and rounding); the table insert/lookup loops are the sequential C file
`pf_table_ref.c` loaded through ctypes.  Pinned against
tests/golden/*.npz, which tests/golden/make_golden.py produced by running the
reference itself (see tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

M64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15          # src/rng.py:16
MIX_M1 = 0xFF51AFD7ED558CCD          # src/rng.py:14
MIX_M2 = 0xC4CEB9FE1A85EC53          # src/rng.py:15
INIT_INDEX = 0x9E3779B97F4A7C15      # src/keys.py:22
INIT_FP = 0xC2B2AE3D27D4EB4F         # src/keys.py:23
EMPTY_TAG = 0xFFFFFFFF00000000       # src/table.py:39
FIXED = 65536                        # src/table.py:38
PRIO_AGE_MASK = 0xFFFFFE             # src/table.py:40
STREAM_ACCUM = 2                     # src/rng.py:20
STREAM_LOOKUP = 3                    # src/rng.py:21
MAX_LEVEL = 31

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "libpf_oracle.so")
_lib = None


# ---------------------------------------------------------------- build / load

def build_lib(force: bool = False) -> str:
    """Compile pf_table_ref.c (gcc, no FMA contraction) into oracle/lib/."""
    src = os.path.join(_HERE, "pf_table_ref.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        vp = ctypes.c_void_p
        lib.orc_accumulate.argtypes = [vp, vp, ctypes.c_int, vp, vp, vp, vp, vp,
                                       ctypes.c_int64, vp, vp, vp, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       vp, vp, vp, vp, vp]
        lib.orc_lookup.argtypes = [vp, ctypes.c_int64, vp, vp, ctypes.c_int64,
                                   ctypes.c_int, vp]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- config

@dataclass
class Config:
    """The FilterConfig knobs the hot path reads (src/keys.py:30-79)."""
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
    sample_cap: int = 256

    @classmethod
    def from_any(cls, cfg) -> "Config":
        fields = cls.__dataclass_fields__
        return cls(**{k: getattr(cfg, k) for k in fields if hasattr(cfg, k)})


# ---------------------------------------------------------------- rng (src/rng.py)

def mix64(x: int) -> int:
    """murmur3 fmix64 on a Python int (src/rng.py:26-34)."""
    x &= M64
    x ^= x >> 33
    x = (x * MIX_M1) & M64
    x ^= x >> 33
    x = (x * MIX_M2) & M64
    x ^= x >> 33
    return x


def mix64_np(x: np.ndarray) -> np.ndarray:
    """Vectorised fmix64 with uint64 wraparound (src/rng.py:51-59)."""
    x = x.astype(np.uint64, copy=True)
    s = np.uint64(33)
    x ^= x >> s
    x *= np.uint64(MIX_M1)
    x ^= x >> s
    x *= np.uint64(MIX_M2)
    x ^= x >> s
    return x


def stream_base(seed: int, stream: int) -> int:
    """h0 = mix64(seed ^ stream*G) (src/rng.py:68)."""
    return mix64((seed & M64) ^ ((stream * GOLDEN) & M64))


def draw_u64(seed: int, stream: int, a, b, c) -> np.ndarray:
    """Counter-based draw (src/rng.py:62-72): absorb a, b, c after h0."""
    g = np.uint64(GOLDEN)
    h = np.uint64(stream_base(seed, stream))
    for f in (a, b, c):
        h = mix64_np(h ^ (np.asarray(f, dtype=np.uint64) + g))
    return h


def draw_unit(seed: int, stream: int, a, b, c) -> np.ndarray:
    """Top 53 bits as a double in [0, 1) (src/rng.py:75-78)."""
    return (draw_u64(seed, stream, a, b, c) >> np.uint64(11)).astype(np.float64) \
        * (1.0 / (1 << 53))


def path_ids(pixel, sample) -> np.ndarray:
    """(sample << 32) | pixel (src/tracer.py:82-84)."""
    return (np.asarray(sample).astype(np.uint64) << np.uint64(32)) \
        | np.asarray(pixel).astype(np.uint64)


def jitter_draws(seed: int, stream: int, pixel, sample):
    """u1, u2 of src/pipeline.py:119-123 (dims 0 and 1, step 0)."""
    pid = path_ids(pixel, sample)
    return draw_unit(seed, stream, pid, 0, 0), draw_unit(seed, stream, pid, 0, 1)


# ---------------------------------------------------------------- keys (src/keys.py)

def lod(distance: np.ndarray, cfg: Config) -> np.ndarray:
    """floor(log2(max(d * C, 1))) clamped to 31 (src/keys.py:245-248)."""
    c_lod = cfg.footprint_scale * cfg.s_pixels / cfg.base_voxel
    ratio = distance * c_lod
    lv = np.floor(np.log2(np.maximum(ratio, 1.0))).astype(np.int64)
    return np.minimum(lv, MAX_LEVEL)


def tangent_frame(n: np.ndarray):
    """Branchless ONB, evaluated left to right (src/keys.py:251-258)."""
    x, y, z = n[:, 0], n[:, 1], n[:, 2]
    s = np.where(z >= 0.0, 1.0, -1.0)
    a = -1.0 / (s + z)
    b = x * y * a
    t1 = np.stack([1.0 + s * x * x * a, s * b, -s * x], axis=1)
    t2 = np.stack([b, s + y * y * a, -y], axis=1)
    return t1, t2


def disc(u1, u2):
    """Polar warp to the radius-1/2 disc (src/keys.py:264-267)."""
    r = 0.5 * np.sqrt(u1)
    phi = (2.0 * math.pi) * u2
    return r * np.cos(phi), r * np.sin(phi)


def voxel_step(level: np.ndarray, cfg: Config) -> np.ndarray:
    return cfg.base_voxel * np.exp2(level.astype(np.float64))


def jitter(pos, nrm, level, u, v, cfg: Config):
    """x + (u t1 + v t2) * step (src/keys.py:261-270)."""
    t1, t2 = tangent_frame(nrm)
    return pos + (u[:, None] * t1 + v[:, None] * t2) * voxel_step(level, cfg)[:, None]


def octa_bins(n: np.ndarray, bins: int) -> np.ndarray:
    """Octahedral normal bin by*bins+bx (src/keys.py:273-283)."""
    s = np.maximum(np.abs(n).sum(axis=1), 1e-300)
    p = n / s[:, None]
    px, py, pz = p[:, 0], p[:, 1], p[:, 2]
    neg = pz < 0.0
    fx = np.where(neg, (1.0 - np.abs(py)) * np.where(px >= 0.0, 1.0, -1.0), px)
    fy = np.where(neg, (1.0 - np.abs(px)) * np.where(py >= 0.0, 1.0, -1.0), py)
    bx = np.minimum(((fx * 0.5 + 0.5) * bins).astype(np.int64), bins - 1)
    by = np.minimum(((fy * 0.5 + 0.5) * bins).astype(np.int64), bins - 1)
    return by * bins + bx


def aux_word(nrm, omega_r, layer, cfg: Config) -> np.ndarray:
    """Normal bin | angle bin << 16 | layer << 24 (src/keys.py:286-299)."""
    aux = np.zeros(len(nrm), np.uint64)
    if cfg.include_normal and not cfg.normal_in_fingerprint:
        aux |= octa_bins(nrm, cfg.normal_bins).astype(np.uint64)
    if cfg.include_incident_angle:
        cos_t = np.clip(np.einsum("ij,ij->i", nrm, omega_r), 0.0, 1.0)
        ab = np.minimum((cos_t * cfg.incident_angle_bins).astype(np.int64),
                        cfg.incident_angle_bins - 1)
        ab = np.where(layer == 1, ab, 0).astype(np.uint64)
        aux |= ab << np.uint64(16)
    if cfg.include_layer:
        aux |= np.asarray(layer).astype(np.uint64) << np.uint64(24)
    return aux


def cell_hashes(qx, qy, qz, level, aux, fp_bins=None):
    """Index hash and fingerprint over (qx,qy,qz,level,aux) (src/keys.py:327-339)."""
    fields = [np.asarray(f).astype(np.uint64) for f in (qx, qy, qz, level, aux)]
    n = len(fields[0])
    h = np.full(n, INIT_INDEX, np.uint64)
    g = np.full(n, INIT_FP, np.uint64)
    for f in fields:
        h = mix64_np(h ^ f)
    for f in fields:
        g = mix64_np(g ^ f)
    fp = ((g ^ (g >> np.uint64(32))) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    if fp_bins is not None:
        fp = (fp << np.uint32(6)) | np.asarray(fp_bins).astype(np.uint32)
    fp = np.where(fp == 0, np.uint32(1), fp)
    return h, fp


@dataclass
class Keys:
    qx: np.ndarray
    qy: np.ndarray
    qz: np.ndarray
    level: np.ndarray
    aux: np.ndarray
    index: np.ndarray
    fingerprint: np.ndarray
    jittered: np.ndarray


def keys(pos, nrm, omega_r, layer, dist, cfg: Config, u=None, v=None,
         level_delta: int = 0) -> Keys:
    """make_key_arrays restated (src/keys.py:342-359); u, v are the disc offsets."""
    lv = np.minimum(lod(dist, cfg) + level_delta, MAX_LEVEL)
    if cfg.jitter and u is not None:
        x = jitter(pos, nrm, lv, u, v, cfg)
        moved = dist + np.linalg.norm(x - pos, axis=1)
        lv = np.minimum(lod(moved, cfg) + level_delta, MAX_LEVEL)
    else:
        x = pos
    q = np.floor(x / voxel_step(lv, cfg)[:, None]).astype(np.int64)
    aux = aux_word(nrm, omega_r, layer, cfg)
    fp_bins = None
    if cfg.include_normal and cfg.normal_in_fingerprint:
        fp_bins = octa_bins(nrm, 8) & 0x3F
    index, fp = cell_hashes(q[:, 0], q[:, 1], q[:, 2], lv, aux, fp_bins)
    return Keys(q[:, 0], q[:, 1], q[:, 2], lv, aux, index, fp, x)


def stream_keys(vs, cfg: Config, seed: int, stream: int = STREAM_ACCUM,
                level_delta: int = 0) -> Keys:
    """vertex_keys restated (src/pipeline.py:126-135)."""
    u = v = None
    if cfg.jitter:
        u1, u2 = jitter_draws(seed, stream, vs.pixel, vs.sample)
        u, v = disc(u1, u2)
    return keys(vs.position, vs.normal, vs.omega_r, vs.layer_id, vs.camera_distance,
                cfg, u, v, level_delta)


# ---------------------------------------------------------------- table (src/table.py)

class Table:
    """Reference VoxelTable state in the reference SoA layout (src/table.py:83-108)."""

    def __init__(self, capacity, probe_limit=32, sum_mode="fixed", evict_horizon=8,
                 evict_min_age=3):
        if capacity < 2 or capacity & (capacity - 1):
            raise ValueError("capacity must be a power of two")
        self.capacity = capacity
        self.probe_limit = probe_limit
        self.sum_mode = sum_mode
        self.evict_horizon = evict_horizon
        self.evict_min_age = evict_min_age
        dt = np.int64 if sum_mode == "fixed" else np.float64
        self.tags = np.full(capacity, EMPTY_TAG, np.uint64)
        self.sums = np.zeros((capacity, 3), dt)
        self.counts = np.zeros(capacity, np.int64)
        self.hist_sums = np.zeros((capacity, 3), dt)
        self.hist_counts = np.zeros(capacity, np.int64)
        self.last_touch = np.zeros(capacity, np.int64)
        self.deltas = np.zeros(capacity, np.float64)
        self.frame = 0
        self.horizon_clears = 0
        self.evictions = 0

    @classmethod
    def from_config(cls, cfg: Config) -> "Table":
        return cls(cfg.capacity, cfg.probe_limit, cfg.sum_mode, cfg.evict_horizon,
                   cfg.evict_min_age)

    def accumulate(self, index, fp, vals, frame):
        """accumulate_batch (src/table.py:117-142) over the C kernel."""
        vals = np.ascontiguousarray(vals, np.float64)
        if np.any(~np.isfinite(vals)) or np.any(vals < 0.0):
            raise ValueError("contributions must be finite and non-negative")
        index = np.ascontiguousarray(index, np.uint64)
        fp = np.ascontiguousarray(fp, np.uint32)
        n = len(index)
        st = np.zeros(n, np.uint8)
        sl = np.full(n, -1, np.int64)
        pl = np.zeros(n, np.uint8)
        vt = np.zeros(n, np.uint64)
        vtt = np.zeros(n, np.int64)
        _load().orc_accumulate(_p(self.tags), _p(self.sums), int(self.sum_mode == "fixed"),
                               _p(self.counts), _p(self.hist_sums), _p(self.hist_counts),
                               _p(self.last_touch), _p(self.deltas), self.capacity,
                               _p(index), _p(fp), _p(vals), n, int(frame),
                               self.probe_limit, self.evict_min_age,
                               _p(st), _p(sl), _p(pl), _p(vt), _p(vtt))
        self.evictions += int((st == 1).sum())
        return st, sl, pl, vt, vtt

    def lookup(self, index, fp):
        index = np.ascontiguousarray(index, np.uint64)
        fp = np.ascontiguousarray(fp, np.uint32)
        out = np.empty(len(index), np.int64)
        _load().orc_lookup(_p(self.tags), self.capacity, _p(index), _p(fp), len(index),
                           self.probe_limit, _p(out))
        return out

    def effective(self, mode, ema_alpha=0.8, delta_max=0.5):
        """Temporally blended (sum, count) per slot (src/table.py:205-238)."""
        if mode == "integrate":
            return self.sums + self.hist_sums, self.counts + self.hist_counts
        live = self.sums.astype(np.float64)
        hist = self.hist_sums.astype(np.float64)
        if self.sum_mode == "fixed":
            live /= FIXED
            hist /= FIXED
        lc = self.counts.astype(np.float64)
        hc = self.hist_counts.astype(np.float64)
        with np.errstate(invalid="ignore", divide="ignore"):
            lmean = np.where(lc[:, None] > 0, live / np.maximum(lc, 1)[:, None], 0.0)
            hmean = np.where(hc[:, None] > 0, hist / np.maximum(hc, 1)[:, None], 0.0)
        if mode == "filter":
            alpha = np.where(hc > 0, np.where(lc > 0, ema_alpha, 1.0), 0.0)
            cnt = lc + hc
        elif mode == "hybrid":
            k = np.clip(self.deltas / delta_max, 0.0, 1.0)
            both = np.maximum(lc + hc, 1.0)
            alpha = np.where(hc > 0, np.where(lc > 0, (1.0 - k) * hc / both, 1.0), 0.0)
            cnt = np.round((1.0 - k) * hc) + lc
        else:
            raise ValueError(f"unknown temporal mode {mode!r}")
        mean = alpha[:, None] * hmean + (1.0 - alpha)[:, None] * lmean
        s = mean * cnt[:, None]
        if self.sum_mode == "fixed":
            s *= FIXED
        return s, cnt

    def begin_frame(self, frame, cfg: Config | None = None):
        """Generation fold, aging, horizon clear (src/table.py:242-298)."""
        mode = cfg.temporal_mode if cfg else "integrate"
        ema = cfg.ema_alpha if cfg else 0.8
        dmax = cfg.delta_max if cfg else 0.5
        cap = cfg.sample_cap if cfg else 0
        occ = self.tags != EMPTY_TAG
        age = frame - self.last_touch
        clear = occ & (age > self.evict_horizon)
        keep = occ & ~clear
        self.horizon_clears += int(clear.sum())
        if mode == "integrate":
            self.hist_sums[keep] += self.sums[keep]
            self.hist_counts[keep] += self.counts[keep]
        else:
            es, ec = self.effective(mode, ema, dmax)
            cnt = np.round(ec).astype(np.int64)
            if mode == "filter":
                cnt = np.minimum(cnt, 1)
            has = keep & (cnt > 0)
            with np.errstate(invalid="ignore", divide="ignore"):
                mean = es / np.maximum(ec, 1e-300)[:, None]
            nh = mean * cnt[:, None]
            if self.sum_mode == "fixed":
                nh = np.floor(nh + 0.5).astype(np.int64)
            self.hist_sums[has] = nh[has]
            self.hist_counts[has] = cnt[has]
            gone = keep & (cnt <= 0)
            self.hist_sums[gone] = 0
            self.hist_counts[gone] = 0
        if cap and mode in ("integrate", "hybrid"):
            over = keep & (self.hist_counts > cap)
            if over.any():
                scale = cap / self.hist_counts[over].astype(np.float64)
                scaled = self.hist_sums[over] * scale[:, None]
                if self.sum_mode == "fixed":
                    scaled = np.floor(scaled + 0.5).astype(np.int64)
                self.hist_sums[over] = scaled
                self.hist_counts[over] = cap
        self.sums[occ] = 0
        self.counts[occ] = 0
        self.deltas[:] = 0.0
        c = np.minimum(self.hist_counts[keep], 255).astype(np.uint64)
        a = np.minimum(age[keep], PRIO_AGE_MASK).astype(np.uint64)
        prio = ((np.uint64(255) - c) << np.uint64(24)) | a
        self.tags[keep] = (prio << np.uint64(32)) | (self.tags[keep] & np.uint64(0xFFFFFFFF))
        self.tags[clear] = EMPTY_TAG
        self.hist_sums[clear] = 0
        self.hist_counts[clear] = 0
        self.last_touch[clear] = 0
        self.frame = frame


# ---------------------------------------------------------------- pipeline (src/pipeline.py)

SOURCE_FINE, SOURCE_NEIGHBORHOOD, SOURCE_COARSE, SOURCE_UNFILTERED = 0, 1, 2, 3


@dataclass
class State:
    fine: Table
    coarse: Table | None

    @classmethod
    def from_config(cls, cfg: Config) -> "State":
        return cls(Table.from_config(cfg),
                   Table.from_config(cfg) if cfg.multi_level else None)


def accumulate_phase(vs, cfg: Config, state: State, frame: int, seed: int):
    """Fine then coarse insert (src/pipeline.py:152-175); returns keys and stats."""
    fk = stream_keys(vs, cfg, seed)
    stats = {"probe_failures": 0, "coarse_probe_failures": 0, "collisions": 0,
             "probe_histogram": {}}
    ck = None
    if len(vs.pixel) == 0:
        return fk, ck, stats
    st, _, pl, _, _ = state.fine.accumulate(fk.index, fk.fingerprint, vs.contribution, frame)
    stats["probe_failures"] = int((st == 2).sum())
    stats["collisions"] = int(pl.astype(np.int64).sum()) - len(vs.pixel)
    hist = np.bincount(pl)
    stats["probe_histogram"] = {int(k): int(v) for k, v in enumerate(hist) if v and k}
    if state.coarse is not None:
        ck = stream_keys(vs, cfg, seed, level_delta=cfg.coarse_delta)
        cst, _, _, _, _ = state.coarse.accumulate(ck.index, ck.fingerprint,
                                                  vs.contribution, frame)
        stats["coarse_probe_failures"] = int((cst == 2).sum())
    return fk, ck, stats


def _rows_mean(sums, cnts, fixed):
    """src/pipeline.py:196-200."""
    d = np.maximum(np.asarray(cnts, np.float64), 1e-300)
    if fixed:
        d = d * 65536.0
    return np.asarray(sums, np.float64) / d[:, None]


def resolve_phase(vs, cfg: Config, state: State, seed: int, spp: int, base_image,
                  fine_keys: Keys | None = None):
    """Fallback ladder and composite (src/pipeline.py:178-283).

    Returns (image, source, chosen)."""
    h, w = base_image.shape[:2]
    n = len(vs.pixel)
    source = np.full(n, SOURCE_UNFILTERED, np.uint8)
    if n == 0:
        return base_image.copy(), source, np.zeros((0, 3))
    lk = stream_keys(vs, cfg, seed, STREAM_LOOKUP) if (cfg.jitter or fine_keys is None) \
        else fine_keys
    fixed = state.fine.sum_mode == "fixed"
    es, ec = state.fine.effective(cfg.temporal_mode, cfg.ema_alpha, cfg.delta_max)
    thr = max(cfg.low_count_threshold, 1)
    chosen = np.array(vs.contribution, np.float64, copy=True)
    slots = state.fine.lookup(lk.index, lk.fingerprint)
    found = slots >= 0
    cnt_f = np.zeros(n, np.float64)
    cnt_f[found] = ec[slots[found]]
    ok_f = cnt_f >= thr

    rest = np.nonzero(~ok_f)[0]
    cnt_n = np.zeros(n, np.float64)
    mean_n = np.zeros((n, 3))
    if len(rest):
        ps = np.zeros((len(rest), 3), es.dtype)
        pc = np.zeros(len(rest), ec.dtype)
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    i2, f2 = cell_hashes(lk.qx[rest] + dx, lk.qy[rest] + dy,
                                         lk.qz[rest] + dz, lk.level[rest], lk.aux[rest])
                    sl = state.fine.lookup(i2, f2)
                    ok = sl >= 0
                    ps[ok] += es[sl[ok]]
                    pc[ok] += ec[sl[ok]]
        cnt_n[rest] = pc
        some = pc > 0
        mean_n[rest[some]] = _rows_mean(ps[some], pc[some], fixed)
    ok_n = ~ok_f & (cnt_n >= thr)

    cnt_c = np.zeros(n, np.float64)
    mean_c = np.zeros((n, 3))
    rest2 = np.nonzero(~ok_f & ~ok_n)[0]
    if len(rest2) and state.coarse is not None:
        sub = _Rows(vs, rest2)
        tag = STREAM_LOOKUP if cfg.jitter else STREAM_ACCUM
        ck = stream_keys(sub, cfg, seed, tag, level_delta=cfg.coarse_delta)
        ces, cec = state.coarse.effective(cfg.temporal_mode, cfg.ema_alpha, cfg.delta_max)
        cs = state.coarse.lookup(ck.index, ck.fingerprint)
        cf = cs >= 0
        rows = rest2[cf]
        cnt_c[rows] = cec[cs[cf]]
        some = cnt_c[rows] > 0
        mean_c[rows[some]] = _rows_mean(ces[cs[cf]][some], cnt_c[rows][some], fixed)
    ok_c = ~ok_f & ~ok_n & (cnt_c >= thr)
    any_n = ~ok_f & ~ok_n & ~ok_c & (cnt_n >= 1)
    any_c = ~ok_f & ~ok_n & ~ok_c & ~any_n & (cnt_c >= 1)

    rows = np.nonzero(ok_f)[0]
    chosen[rows] = _rows_mean(es[slots[rows]], cnt_f[rows], fixed)
    source[rows] = SOURCE_FINE
    for m, mean, code in ((ok_n | any_n, mean_n, SOURCE_NEIGHBORHOOD),
                          (ok_c | any_c, mean_c, SOURCE_COARSE)):
        rows = np.nonzero(m)[0]
        chosen[rows] = mean[rows]
        source[rows] = code
    flat = np.zeros((h * w, 3))
    np.add.at(flat, vs.pixel, vs.throughput * chosen)
    image = base_image + flat.reshape(h, w, 3) / spp
    return image, source, chosen


class _Rows:
    """Row subset of a vertex stream (the reference's VertexStream.select)."""

    def __init__(self, vs, rows):
        for f in ("position", "normal", "omega_r", "contribution", "throughput",
                  "pixel", "sample", "layer_id", "camera_distance"):
            setattr(self, f, getattr(vs, f)[rows])


def filter_frame(vs, cfg: Config, state: State, frame: int, seed: int, spp: int,
                 base_image):
    """begin_frame on both tables, accumulate, resolve (src/pipeline.py:331-344
    without the tracer)."""
    state.fine.begin_frame(frame, cfg)
    if state.coarse is not None:
        state.coarse.begin_frame(frame, cfg)
    fk, ck, stats = accumulate_phase(vs, cfg, state, frame, seed)
    image, source, chosen = resolve_phase(vs, cfg, state, seed, spp, base_image, fk)
    return image, source, chosen, stats
