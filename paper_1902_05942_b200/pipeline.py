"""Per-frame filter orchestration on the device (src/pipeline.py, tracer excluded).

accumulate_phase launches ONE fused kernel per frame (keys for the fine and coarse
tables + warp-merged inserts); resolve_phase launches the fine-rung kernel, the
fallback kernel over the compacted low-count rows and the image finalisation.
Nothing synchronises with the host until a statistic or host array is read.

Ladder (src/pipeline.py:1-15): fine voxel >= threshold -> 3x3x3 neighbourhood ->
coarse voxel -> any neighbourhood / coarse samples -> unfiltered contribution.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import math

import numpy as np
import torch

from . import _lib, rng
from .keys import FilterConfig, KeyArrays, _empty_keys, _key_out, as_f64, as_i64, device, \
    vertices_c
from .table import EvictionEvent, VoxelTable, _AGE_MASK

SOURCE_FINE = 0
SOURCE_NEIGHBORHOOD = 1
SOURCE_COARSE = 2
SOURCE_UNFILTERED = 3

_FIELDS = ("position", "normal", "omega_r", "contribution", "throughput", "pixel", "sample",
           "layer_id", "camera_distance")


@dataclass
class VertexDescriptor:
    """One recorded path vertex, the scalar view of a stream row (src/tracer.py:46-62),
    with numpy vectors and Python scalars as in the reference."""

    position: np.ndarray
    normal: np.ndarray
    omega_r: np.ndarray
    contribution: np.ndarray
    throughput: np.ndarray
    pixel: int
    sample: int
    layer_id: int
    camera_distance: float

    @property
    def path_id(self) -> int:
        return (self.sample << 32) | self.pixel


@dataclass
class VertexStream:
    """Struct-of-arrays vertex record (src/tracer.py:66-104) as CUDA tensors."""

    position: torch.Tensor
    normal: torch.Tensor
    omega_r: torch.Tensor
    contribution: torch.Tensor
    throughput: torch.Tensor
    pixel: torch.Tensor
    sample: torch.Tensor
    layer_id: torch.Tensor
    camera_distance: torch.Tensor

    def __len__(self) -> int:
        return int(self.pixel.shape[0])

    @property
    def path_id(self) -> torch.Tensor:
        return (self.sample << 32) | self.pixel

    @classmethod
    def from_any(cls, vs) -> "VertexStream":
        """Upload a reference VertexStream (numpy fields) or pass a device one through."""
        if isinstance(vs, cls):
            return vs
        vec = {"position", "normal", "omega_r", "contribution", "throughput"}
        return cls(**{f: (as_f64(getattr(vs, f), 3) if f in vec else
                          as_f64(getattr(vs, f)).reshape(-1) if f == "camera_distance" else
                          as_i64(getattr(vs, f)).reshape(-1)) for f in _FIELDS})

    def select(self, rows) -> "VertexStream":
        """Rows by index array or boolean mask (src/tracer.py:92-93)."""
        if isinstance(rows, torch.Tensor) and rows.dtype == torch.bool:
            r = rows.to(self.pixel.device)
        elif not isinstance(rows, torch.Tensor) and np.asarray(rows).dtype == np.bool_:
            r = torch.as_tensor(np.asarray(rows), device=self.pixel.device)
        else:
            r = as_i64(rows).reshape(-1)
        return VertexStream(*(getattr(self, f)[r] for f in _FIELDS))

    def descriptor(self, i: int) -> VertexDescriptor:
        """Row i as a host VertexDescriptor (src/tracer.py:86-90); one device read."""
        row = [getattr(self, f)[i].cpu().numpy() for f in _FIELDS]
        return VertexDescriptor(*row[:5], int(row[5]), int(row[6]), int(row[7]), float(row[8]))

    @staticmethod
    def concat(streams: list) -> "VertexStream":
        """Row concatenation (src/tracer.py:95-101); an empty list gives an empty stream."""
        if not streams:
            return VertexStream.empty()
        return VertexStream(*(torch.cat([getattr(VertexStream.from_any(s), f) for s in streams])
                              for f in _FIELDS))

    @staticmethod
    def empty() -> "VertexStream":
        dev = device()
        e3 = torch.zeros((0, 3), dtype=torch.float64, device=dev)
        e1 = torch.zeros(0, dtype=torch.int64, device=dev)
        return VertexStream(e3, e3, e3, e3, e3, e1, e1, e1, e1.to(torch.float64))

    def numpy(self):
        """Host copy with the reference's field dtypes (a SimpleNamespace of arrays)."""
        from types import SimpleNamespace
        return SimpleNamespace(**{f: getattr(self, f).cpu().numpy() for f in _FIELDS})

    def c_struct(self):
        """pf_vertices view, cached while the field tensors stay the same objects."""
        key = tuple(id(getattr(self, f)) for f in _FIELDS)
        cached = self.__dict__.get("_c_cache")
        if cached is not None and cached[0] == key:
            return cached[1]
        c = vertices_c(self.position, self.normal, self.omega_r, self.layer_id,
                       self.camera_distance, pixel=self.pixel, sample=self.sample,
                       contribution=self.contribution, throughput=self.throughput)
        self.__dict__["_c_cache"] = (key, c)
        return c


@dataclass
class ResolveReport:
    source: torch.Tensor
    image: torch.Tensor
    means: torch.Tensor | None = None

    @property
    def counts(self) -> dict[str, int]:
        c = torch.bincount(self.source.to(torch.int64), minlength=4).cpu().numpy()
        return {"fine_voxel": int(c[0]), "neighborhood": int(c[1]),
                "coarse_voxel": int(c[2]), "unfiltered": int(c[3])}


class FrameStats:
    """Frame statistics (src/pipeline.py:51-85) backed by a device counter array;
    values synchronise on first read."""

    _SCALARS = ("frame", "n_vertices", "probe_failures", "coarse_probe_failures", "collisions",
                "evictions", "horizon_clears", "occupancy_fine", "occupancy_coarse",
                "time_trace", "time_accumulate", "time_resolve", "time_total")

    def __init__(self, frame: int = 0, n_vertices: int = 0, counters: torch.Tensor | None = None):
        self.frame = frame
        self.n_vertices = n_vertices
        self.counters = counters
        self._host = None
        self.evictions = 0
        self.horizon_clears = 0
        self.occupancy_fine = 0.0
        self.occupancy_coarse = 0.0
        self.source_counts: dict[str, int] = {}
        self.time_trace = 0.0
        self.time_accumulate = 0.0
        self.time_resolve = 0.0
        self.time_total = 0.0

    def _c(self) -> np.ndarray:
        if self._host is None:
            self._host = (self.counters.cpu().numpy() if self.counters is not None
                          else np.zeros(_lib.STAT_COUNT, np.int64))
        return self._host

    @property
    def probe_failures(self) -> int:
        return int(self._c()[_lib.STAT_PROBE_FAILURES])

    @property
    def coarse_probe_failures(self) -> int:
        return int(self._c()[_lib.STAT_COARSE_PROBE_FAILURES])

    @property
    def collisions(self) -> int:
        return int(self._c()[_lib.STAT_PROBE_LEN_SUM]) - self.n_vertices if self.n_vertices else 0

    @property
    def probe_histogram(self) -> dict[int, int]:
        h = self._c()[_lib.STAT_HIST_BASE:_lib.STAT_HIST_BASE + 256]
        return {int(k): int(v) for k, v in enumerate(h) if v and k}

    def lines(self) -> list[str]:
        out = [f"frame={self.frame}", f"vertices={self.n_vertices}",
               f"probe_failures={self.probe_failures}",
               f"coarse_probe_failures={self.coarse_probe_failures}",
               f"collisions={self.collisions}", f"evictions={self.evictions}",
               f"horizon_clears={self.horizon_clears}",
               f"occupancy_fine={self.occupancy_fine:.6f}",
               f"occupancy_coarse={self.occupancy_coarse:.6f}"]
        for k in sorted(self.probe_histogram):
            out.append(f"probe_hist_{k}={self.probe_histogram[k]}")
        for k, v in self.source_counts.items():
            out.append(f"source_{k}={v}")
        out += [f"time_trace={self.time_trace:.6f}", f"time_accumulate={self.time_accumulate:.6f}",
                f"time_resolve={self.time_resolve:.6f}", f"time_total={self.time_total:.6f}"]
        return out


@dataclass
class FrameState:
    """Persistent fine/coarse tables (src/pipeline.py:88-105)."""

    fine: VoxelTable
    coarse: VoxelTable | None
    frame: int = 0
    prev_fine_keys: KeyArrays | None = None
    prev_coarse_keys: KeyArrays | None = None
    prev_seed: int = 0
    prev_spp: int = 0
    scratch: dict = field(default_factory=dict)
    lookup_keys: tuple | None = None
    pending_validation: list = field(default_factory=list)
    prev_vertices: object = None  # last rendered frame's VertexStream (hybrid replay)

    def poll_validation(self, wait: bool = False, parity: int | None = None):
        """Raise for a frame whose device input check failed (its kernels were guarded:
        the tables are untouched).  Non-blocking for landed flags; waits for all flags
        when wait=True and for the flag of `parity` (its pinned slot is about to be
        reused)."""
        keep = []
        bad = None
        for host, done, frame, par in self.pending_validation:
            if wait or par == parity or done.query():
                done.synchronize()
                if int(host[0]) and bad is None:
                    bad = frame
            else:
                keep.append((host, done, frame, par))
        self.pending_validation = keep
        if bad is not None:
            raise ValueError(f"frame {bad}: contributions must be finite and non-negative "
                             "(the frame was rejected; tables unchanged)")

    def drain_events(self, parity: int):
        """Move the eviction records still held in the event buffer of this parity
        (written two frames ago) into the table's log before the buffer is reused."""
        self.fine._drain_tag(parity)

    def pinned_count(self, parity: int) -> torch.Tensor:
        key = f"_pinned_count{parity}"
        p = self.scratch.get(key)
        if p is None:
            p = torch.zeros(1, dtype=torch.int64).pin_memory()
            self.scratch[key] = p
        return p

    @classmethod
    def from_config(cls, cfg: FilterConfig, backend: str | None = None,
                    ordered: bool = False) -> "FrameState":
        _lib.configure_l2()
        fine = VoxelTable.from_config(cfg, backend, ordered)
        coarse = VoxelTable.from_config(cfg, backend, ordered) if cfg.multi_level else None
        return cls(fine, coarse)

    def buffer(self, name: str, shape, dtype) -> torch.Tensor:
        """Reusable device scratch (caching allocator friendly, no per-frame memsets).
        The shaped view is cached too: a frame asks for the same nine buffers each call."""
        shape = tuple(int(d) for d in shape) if isinstance(shape, (tuple, list)) else (int(shape),)
        views = self.scratch.setdefault("_views", {})
        hit = views.get(name)
        if hit is not None and hit[0] == shape and hit[1] == dtype and \
                hit[2] is self.scratch.get(name):
            return hit[3]
        n = math.prod(shape)
        b = self.scratch.get(name)
        if b is None or b.numel() < n or b.dtype != dtype:
            b = torch.empty(max(n, 1), dtype=dtype, device=device())
            self.scratch[name] = b
        v = b[:n].view(*shape) if n else b[:0]
        views[name] = (shape, dtype, b, v)
        return v


class LazyKeyArrays:
    """KeyArrays that are only materialised (one key-kernel launch) when read.

    accumulate_phase returns these: the fused insert kernel never writes per-vertex
    keys to HBM, yet the reference API (src/pipeline.py:175) hands keys back."""

    def __init__(self, vs: VertexStream, cfg: FilterConfig, seed: int, stream_tag: int,
                 level_delta: int):
        self._args = (vs, cfg, seed, stream_tag, level_delta)
        self._keys: KeyArrays | None = None

    def materialize(self) -> KeyArrays:
        if self._keys is None:
            self._keys = vertex_keys(*self._args)
        return self._keys

    def __len__(self):
        return len(self._args[0])

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.materialize(), name)


def vertex_keys(vertices, cfg: FilterConfig, seed: int,
                stream_tag: int = rng.STREAM_JITTER_ACCUM, level_delta: int = 0) -> KeyArrays:
    """Key arrays of a vertex stream with the given jitter stream (src/pipeline.py:126-135)."""
    vs = VertexStream.from_any(vertices)
    n = len(vs)
    out = _empty_keys(n)
    if n == 0:
        return out
    v, keep = vs.c_struct()
    ko = _key_out(out)
    _lib.call("pf_vertex_keys", ctypes.byref(cfg.to_c()), ctypes.byref(v),
              rng.stream_base(seed, stream_tag), int(level_delta), ctypes.byref(ko),
              _lib.stream_handle())
    del keep
    return out


def check_contributions(vals: torch.Tensor, flag: torch.Tensor, wait: bool = True):
    """accumulate_batch's input check (src/table.py:127-129) as one device pass; with
    wait=False the caller launches flag-guarded work first and calls raise_if_bad."""
    flag.zero_()
    _lib.call("pf_check_contributions", vals.data_ptr(), int(vals.numel()), flag.data_ptr(),
              _lib.stream_handle())
    if wait:
        raise_if_bad(flag)


def raise_if_bad(flag: torch.Tensor):
    if int(flag.item()):
        raise ValueError("contributions must be finite and non-negative")


def accumulate_phase(vertices, cfg: FilterConfig, state: FrameState, frame: int, seed: int,
                     threads: int = 1, validate: bool = True):
    """Insert all vertices into the fine and coarse tables (src/pipeline.py:152-175).

    Returns (fine keys, coarse keys, stats); keys are lazy (computed on first read)."""
    vs = VertexStream.from_any(vertices)
    n = len(vs)
    parity = int(frame) & 1
    state.drain_events(parity)  # this parity's event log buffer is about to be reused
    counters = torch.zeros(_lib.STAT_COUNT, dtype=torch.int64, device=vs.pixel.device)
    stats = FrameStats(frame=frame, n_vertices=n, counters=counters)
    fine_keys = LazyKeyArrays(vs, cfg, seed, rng.STREAM_JITTER_ACCUM, 0)
    coarse_keys = None
    if n == 0:
        return fine_keys, coarse_keys, stats
    if state.coarse is not None:
        coarse_keys = LazyKeyArrays(vs, cfg, seed, rng.STREAM_JITTER_ACCUM, cfg.coarse_delta)
    if state.fine.ordered:
        if validate:
            check_contributions(vs.contribution, state.buffer("bad_flag", (1,), torch.int32))
        return _accumulate_ordered(vs, cfg, state, frame, seed, stats, fine_keys, coarse_keys)
    flag = None
    if validate:
        # check, then the flag-guarded insert (no mutation on bad input), then one sync
        flag = state.buffer("bad_flag", (1,), torch.int32)
        check_contributions(vs.contribution, flag, wait=False)
    lk_keys = state.buffer("lk_keys", (n,), torch.int64)  # packed fp << 32 | slot index
    lookup_seed = rng.stream_base(seed, rng.STREAM_JITTER_LOOKUP)
    events = state.buffer(f"events{parity}", (n, 4), torch.int64)
    ev_count = state.buffer(f"event_count{parity}", (1,), torch.int64)
    ev_count.zero_()
    v, keep = vs.c_struct()
    ft = state.fine.c_table()
    ct = state.coarse.c_table() if state.coarse is not None else None
    _lib.call("pf_insert_frame", ctypes.byref(cfg.to_c()), ctypes.byref(v), ctypes.byref(ft),
              ctypes.byref(ct) if ct is not None else None,
              rng.stream_base(seed, rng.STREAM_JITTER_ACCUM), int(frame), counters.data_ptr(),
              events.data_ptr(), ev_count.data_ptr(), n, _lib.ptr(flag), lookup_seed,
              lk_keys.data_ptr(), _lib.stream_handle())
    del keep
    # resolve_phase reuses these lookup keys when called for the same stream / seed / knobs
    state.lookup_keys = (vs, lookup_seed, cfg.to_c(), lk_keys)
    _register_event_drain(state, frame, events, ev_count, parity)
    if flag is not None:
        raise_if_bad(flag)  # the guarded kernel left the tables untouched
    return fine_keys, coarse_keys, stats


def _register_event_drain(state: FrameState, frame: int, events: torch.Tensor,
                          ev_count: torch.Tensor, parity: int) -> torch.cuda.Event:
    """Queue the eviction log of this frame: its count goes to pinned host memory
    without a sync; the rows are read before the device buffer (one of two, by frame
    parity) is reused two frames later.  Returns the event that marks the copy (and
    every copy queued before it) landed."""
    host = state.pinned_count(parity)
    host.copy_(ev_count, non_blocking=True)
    done = torch.cuda.Event()
    done.record()
    pending = {"drained": False}

    def drain(frame=frame, events=events, host=host, done=done, pending=pending):
        if pending["drained"]:
            return []
        pending["drained"] = True
        done.synchronize()
        k = int(host[0])
        if k == 0:
            return []
        rows = events[:k].cpu().numpy()
        rows = rows[np.argsort(rows[:, 0], kind="stable")]
        out = []
        for _, slot, vtag, vtouch in rows:
            age = (int(np.int64(vtag).view(np.uint64)) >> 32) & _AGE_MASK
            out.append(EvictionEvent(frame, int(slot), age, int(vtouch)))
        return out

    state.fine._add_pending_events(drain, parity)
    return done


def _accumulate_ordered(vs, cfg, state, frame, seed, stats, fine_keys, coarse_keys):
    """Sequential-order variant (tables created with ordered=True): materialise keys,
    then the in-order batch insert, reproducing the reference's threads=1 layout."""
    c = stats.counters
    fk = fine_keys.materialize()
    st, _, pl = state.fine.accumulate_batch(fk.index, fk.fingerprint, vs.contribution, frame)
    c[_lib.STAT_PROBE_FAILURES] = (st == 2).sum()
    c[_lib.STAT_EVICTIONS] = (st == 1).sum()
    pl64 = pl.to(torch.int64)
    c[_lib.STAT_PROBE_LEN_SUM] = pl64.sum()
    c[_lib.STAT_HIST_BASE:_lib.STAT_HIST_BASE + 256] += torch.bincount(pl64, minlength=256)[:256]
    if state.coarse is not None:
        ck = coarse_keys.materialize()
        cst, _, _ = state.coarse.accumulate_batch(ck.index, ck.fingerprint, vs.contribution, frame)
        c[_lib.STAT_COARSE_PROBE_FAILURES] = (cst == 2).sum()
        c[_lib.STAT_COARSE_EVICTIONS] = (cst == 1).sum()
    return fine_keys, coarse_keys, stats


def resolve_phase(vertices, cfg: FilterConfig, state: FrameState, frame: int, seed: int,
                  spp: int, base_image, fine_keys=None, want_means: bool = True):
    """Per-vertex filtered means composited onto the base image (src/pipeline.py:207-283).

    Returns (image, ResolveReport) as device tensors.  With jitter disabled the
    lookup keys equal the accumulate keys, which the kernel recomputes in registers
    instead of reading `fine_keys` back from HBM."""
    vs = VertexStream.from_any(vertices)
    base = as_f64(base_image)
    h, w = int(base.shape[0]), int(base.shape[1])
    n = len(vs)
    dev = base.device
    source = torch.empty(n, dtype=torch.uint8, device=dev)
    chosen = torch.empty((n, 3), dtype=torch.float64, device=dev) if want_means else None
    image = torch.empty_like(base)
    flat = state.buffer("flat", (h * w, 3), torch.float64)
    work = state.buffer("work", (_lib.work_rows(n),), torch.int64)
    work_count = state.buffer("work_count", (_lib.WORK_LISTS,), torch.int64)
    counters = torch.zeros(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
    v, keep = vs.c_struct()
    ft = state.fine.c_table()
    ct = state.coarse.c_table() if state.coarse is not None else None
    coarse_tag = rng.STREAM_JITTER_LOOKUP if cfg.jitter else rng.STREAM_JITTER_ACCUM
    lookup_seed = rng.stream_base(seed, rng.STREAM_JITTER_LOOKUP)
    cc = cfg.to_c()
    lk = state.lookup_keys
    lk_ok = lk is not None and lk[0] is vs and lk[1] == lookup_seed and lk[2] is cc
    _lib.call("pf_resolve_frame", ctypes.byref(cc), ctypes.byref(v), ctypes.byref(ft),
              ctypes.byref(ct) if ct is not None else None,
              lookup_seed, rng.stream_base(seed, coarse_tag),
              int(spp), base.data_ptr(), h * w, image.data_ptr(), flat.data_ptr(),
              work.data_ptr(), work_count.data_ptr(), source.data_ptr(), _lib.ptr(chosen),
              counters.data_ptr(), lk[3].data_ptr() if lk_ok else None,
              state.buffer("eff_records", (state.fine.capacity, 4), torch.int64).data_ptr(),
              state.buffer("fallback_keys", (max(n, 1), 8), torch.int64).data_ptr(),
              _lib.stream_handle())
    del keep
    report = ResolveReport(source, image, chosen)
    report.counters = counters
    return image, report


def _table_key(t: VoxelTable):
    """Changes whenever the table may have changed: a C call on it (c_table), or an
    in-place torch write to any of its storages (tensor version counters)."""
    return (t.tags.data_ptr(), t.__dict__.get("_c_calls", 0), t.tags._version,
            t.counts._version, t._sums._version, t._cold._version)


def _occ_key(state: FrameState):
    return (_table_key(state.fine), _table_key(state.coarse) if state.coarse is not None else None)


def _fused_frame(vs: VertexStream, base_image, cfg: FilterConfig, state: FrameState, frame: int,
                 spp: int, seed: int, validate: bool, want_means: bool, phase_events=None):
    n = len(vs)
    base = as_f64(base_image)
    h, w = int(base.shape[0]), int(base.shape[1])
    dev = base.device
    parity = int(frame) & 1
    state.drain_events(parity)
    state.poll_validation(parity=parity)  # surface a rejected earlier frame
    acc = torch.empty(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
    res = torch.empty(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
    source = torch.empty(n, dtype=torch.uint8, device=dev)
    chosen = torch.empty((n, 3), dtype=torch.float64, device=dev) if want_means else None
    image = torch.empty_like(base)
    events = state.buffer(f"events{parity}", (max(n, 1), 4), torch.int64)
    ev_count = state.buffer(f"event_count{parity}", (1,), torch.int64)
    flag = state.buffer("bad_flag", (1,), torch.int32) if validate else None
    lk_keys = state.buffer("lk_keys", (max(n, 1),), torch.int64)
    b = _lib.PfFrameBuffers()
    b.acc_stats, b.res_stats = acc.data_ptr(), res.data_ptr()
    b.events, b.event_count, b.event_capacity = events.data_ptr(), ev_count.data_ptr(), n
    b.bad_flag = _lib.ptr(flag)
    b.horizon_clears_fine = state.fine._clears.data_ptr()
    b.horizon_clears_coarse = state.coarse._clears.data_ptr() if state.coarse is not None else None
    b.lookup_keys = lk_keys.data_ptr()
    b.eff_records = state.buffer("eff_records", (state.fine.capacity, 4), torch.int64).data_ptr()
    b.flat = state.buffer("flat", (h * w, 3), torch.float64).data_ptr()
    b.work = state.buffer("work", (_lib.work_rows(n),), torch.int64).data_ptr()
    b.work_count = state.buffer("work_count", (_lib.WORK_LISTS,), torch.int64).data_ptr()
    b.fallback_keys = state.buffer("fallback_keys", (max(n, 1), 8), torch.int64).data_ptr()
    if phase_events is not None:  # torch.cuda.Events recorded inside the C call
        for k, e in enumerate(phase_events):
            b.phase_events[k] = e.cuda_event
    # occupied-slot lists: the frame writes the slots occupied at its end into one of two
    # list buffers; the next frame's begin_frame folds exactly those slots (no tag sweep)
    # if nothing touched the tables in between (same key), else it sweeps
    prev = state.scratch.get("_occ_prev")
    use_in = prev is not None and prev[0] == _occ_key(state)
    out_idx = 1 - prev[1] if prev is not None else 0
    cap_c = state.coarse.capacity if state.coarse is not None else 1

    def occ_bufs(i):
        return (state.buffer(f"occ_fine{i}", (state.fine.capacity,), torch.int32),
                state.buffer(f"occ_coarse{i}", (cap_c,), torch.int32),
                state.buffer(f"occ_n{i}", (2,), torch.int64))
    of, oc, on = occ_bufs(out_idx)
    b.occ_out[0], b.occ_out[1], b.occ_count_out = of.data_ptr(), oc.data_ptr(), on.data_ptr()
    if use_in:
        inf, inc, inn = occ_bufs(prev[1])
        b.occ_in[0], b.occ_in[1], b.occ_count_in = inf.data_ptr(), inc.data_ptr(), inn.data_ptr()
    v, keep = vs.c_struct()
    ft = state.fine.c_table()
    ct = state.coarse.c_table() if state.coarse is not None else None
    cc = cfg.to_c()
    lookup_seed = rng.stream_base(seed, rng.STREAM_JITTER_LOOKUP)
    coarse_tag = rng.STREAM_JITTER_LOOKUP if cfg.jitter else rng.STREAM_JITTER_ACCUM
    _lib.call("pf_filter_frame", ctypes.byref(cc), ctypes.byref(v), ctypes.byref(ft),
              ctypes.byref(ct) if ct is not None else None, int(frame),
              rng.stream_base(seed, rng.STREAM_JITTER_ACCUM), lookup_seed,
              rng.stream_base(seed, coarse_tag), int(spp), base.data_ptr(), h * w,
              image.data_ptr(), source.data_ptr(), _lib.ptr(chosen), ctypes.byref(b),
              _lib.stream_handle())
    del keep
    # the lists describe the tables as this call left them (none without an effective sweep)
    if n:
        state.scratch["_occ_prev"] = (_occ_key(state), out_idx)
    else:
        state.scratch.pop("_occ_prev", None)
    state.fine.frame = frame
    if state.coarse is not None:
        state.coarse.frame = frame
    state.lookup_keys = (vs, lookup_seed, cc, lk_keys[:n])
    stats = FrameStats(frame=frame, n_vertices=n, counters=acc)
    report = ResolveReport(source, image, chosen)
    report.counters = res
    fine_keys = LazyKeyArrays(vs, cfg, seed, rng.STREAM_JITTER_ACCUM, 0)
    coarse_keys = (LazyKeyArrays(vs, cfg, seed, rng.STREAM_JITTER_ACCUM, cfg.coarse_delta)
                   if state.coarse is not None else None)
    flag_host = None
    if flag is not None and n and validate != "sync":
        # deferred: queue the flag read, raise when it has landed (the eviction count's
        # event below marks both copies)
        key = f"_pinned_flag{parity}"
        if key not in state.scratch:
            state.scratch[key] = torch.empty(1, dtype=torch.int32).pin_memory()
        flag_host = state.scratch[key]
        flag_host.copy_(flag, non_blocking=True)
    if n:
        done = _register_event_drain(state, frame, events, ev_count, parity)
        if flag_host is not None:
            state.pending_validation.append((flag_host, done, frame, parity))
    if flag is not None and n and validate == "sync":
        raise_if_bad(flag)
    return image, report, stats, fine_keys, coarse_keys


def filter_frame(vertices, base_image, cfg: FilterConfig, state: FrameState, spp: int,
                 seed: int, validate: bool = True, want_means: bool = True, phase_events=None):
    """One frame of the filter without the tracer: begin_frame on both tables,
    accumulate, resolve (src/pipeline.py:321-363 minus trace/hybrid replay).

    Parallel-insert tables run the whole frame as ONE C-ABI call (pf_filter_frame):
    every kernel is queued back to back on the current stream; the only host sync is
    the input-check flag read at the end (validate=True), after which a ValueError
    means the guarded kernels left the tables untouched."""
    frame = state.frame
    vs = VertexStream.from_any(vertices)  # upload once for both phases
    if state.fine.ordered:
        state.fine.begin_frame(frame, cfg)
        if state.coarse is not None:
            state.coarse.begin_frame(frame, cfg)
        fine_keys, coarse_keys, stats = accumulate_phase(vs, cfg, state, frame, seed,
                                                         validate=validate)
        image, report = resolve_phase(vs, cfg, state, frame, seed, spp, base_image, fine_keys,
                                      want_means=want_means)
    else:
        image, report, stats, fine_keys, coarse_keys = _fused_frame(
            vs, base_image, cfg, state, frame, spp, seed, validate, want_means, phase_events)
    state.prev_fine_keys = fine_keys
    state.prev_coarse_keys = coarse_keys
    state.prev_seed = seed
    state.prev_spp = spp
    state.frame = frame + 1
    return image, report, stats
