"""Device-resident voxel table (src/table.py) over the sm_100a table kernels.

The reference's fields (src/table.py:96-103), with the same values and dtypes:

    tags        u64[C]   (stored in an int64 tensor)  prio<<56 | age<<32 | fingerprint
    sums        i64|f64[C,3]   live generation radiance (16.16 fixed point or float)
    counts      i64[C]
    hist_sums   i64|f64[C,3]   previous generations
    hist_counts i64[C]
    last_touch  i64[C]
    deltas      f64[C]

Layout in HBM (include/pathfilter_b200.h, pf_table): `tags` and `counts` dense, the
live `sums` channel-major ([3][C]: a vertex's three radiance REDs go to three lines, which
the L2 atomic units serve in parallel -- the reference's [C][3] rows put them on one line,
and every per-slot record layout tried, where the count shares the sums' line, was
slower still), and the fields only the per-frame sweeps read in one 64-byte cold record
per slot (last_touch, hist_count, delta, pad, hist_sums[3], pad).  The attributes above
are strided views; `state()` / `dump()` export the reference's SoA arrays.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .keys import CellHashes, FilterConfig, as_f64, as_i64, as_u32_bits, device, temporal_code, \
    u64_numpy

FIXED_SCALE = 65536
EMPTY_TAG = 0xFFFFFFFF00000000
EMPTY_TAG_I64 = EMPTY_TAG - (1 << 64)
_AGE_MASK = 0xFFFFFE
_DUMP_MAGIC = b"PFVT\x01"
COLD_WORDS = 8   # 64-bit words per slot cold record (include/pathfilter_b200.h, pf_table)


def quantize_fixed(values) -> np.ndarray:
    """16.16 fixed point, half up (src/table.py:44-46); host helper for tests/exports."""
    return np.floor(np.asarray(values, np.float64) * FIXED_SCALE + 0.5).astype(np.int64)


def fixed_to_float(sums) -> np.ndarray:
    return np.asarray(sums, np.float64) / FIXED_SCALE


def pack_priority(count, age):
    """Priority word (src/table.py:53-57); smaller values win."""
    c = np.minimum(count, 255).astype(np.uint64)
    a = np.minimum(age, _AGE_MASK).astype(np.uint64)
    return ((np.uint64(255) - c) << np.uint64(24)) | a


class Outcome(Enum):
    ACCUMULATED = 0
    EVICTED_THEN_ACCUMULATED = 1
    PROBE_LIMIT_EXCEEDED = 2


@dataclass
class InsertOutcome:
    status: Outcome
    slot: int


@dataclass
class EvictionEvent:
    frame: int
    slot: int
    victim_age: int
    victim_last_touch: int


class VoxelTable:
    """One resolution level of the filter cache (src/table.py:80-340), in HBM."""

    def __init__(self, capacity: int, probe_limit: int = 32, sum_mode: str = "fixed",
                 evict_horizon: int = 8, evict_min_age: int = 3, backend: str | None = None,
                 ordered: bool = False):
        if capacity < 2 or capacity & (capacity - 1):
            raise ValueError("capacity must be a power of two")
        if sum_mode not in ("fixed", "float"):
            raise ValueError(f"unknown sum_mode {sum_mode!r}")
        dev = device()
        self.capacity = int(capacity)
        self.probe_limit = int(probe_limit)
        self.sum_mode = sum_mode
        self.evict_horizon = int(evict_horizon)
        self.evict_min_age = int(evict_min_age)
        # ordered=True reproduces the reference's sequential slot layout exactly
        self.ordered = bool(ordered)
        self.tags = torch.full((capacity,), EMPTY_TAG_I64, dtype=torch.int64, device=dev)
        z = lambda *shape: torch.zeros(shape, dtype=torch.int64, device=dev)  # noqa: E731
        as_sum = (lambda x: x) if sum_mode == "fixed" else (lambda x: x.view(torch.float64))
        # dense tags and counts, channel-major live sums, one 64-byte cold record per slot
        # (include/pathfilter_b200.h, pf_table); the attributes are views
        self.counts = z(capacity)
        self._sums = z(3, capacity)
        self.sums = as_sum(self._sums.t())
        self._cold = z(capacity, COLD_WORDS)
        c = self._cold
        self.last_touch, self.hist_counts = c[:, 0], c[:, 1]
        self.deltas = c[:, 2].view(torch.float64)
        self.hist_sums = as_sum(c[:, 4:7])
        self.frame = 0
        self._events: list[EvictionEvent] = []
        self._pending_events: list = []
        self._clears = torch.zeros(1, dtype=torch.int64, device=dev)
        self.shadow: dict[int, set] | None = None

    @classmethod
    def from_config(cls, cfg: FilterConfig, backend: str | None = None,
                    ordered: bool = False) -> "VoxelTable":
        return cls(cfg.capacity, cfg.probe_limit, cfg.sum_mode, cfg.evict_horizon,
                   cfg.evict_min_age, backend, ordered)

    # -- C view ---------------------------------------------------------------

    def c_table(self) -> _lib.PfTable:
        # every C call that may write the table goes through here: the count lets a frame
        # know the table is exactly as the previous frame left it (pipeline._occ_key)
        self.__dict__["_c_calls"] = self.__dict__.get("_c_calls", 0) + 1
        key = (self.tags.data_ptr(), self.probe_limit, self.evict_min_age, self.evict_horizon)
        cached = self.__dict__.get("_c_cache")
        if cached is not None and cached[0] == key:
            return cached[1]
        t = self._build_c()
        self.__dict__["_c_cache"] = (key, t)
        return t

    def _build_c(self) -> _lib.PfTable:
        t = _lib.PfTable()
        t.tags = self.tags.data_ptr()
        t.sums = self.sums.data_ptr()
        t.counts = self.counts.data_ptr()
        t.hist_sums = self.hist_sums.data_ptr()
        t.hist_counts = self.hist_counts.data_ptr()
        t.last_touch = self.last_touch.data_ptr()
        t.deltas = self.deltas.data_ptr()
        t.capacity = self.capacity
        t.sum_mode = 0 if self.sum_mode == "fixed" else 1
        t.probe_limit = self.probe_limit
        t.evict_min_age = self.evict_min_age
        t.evict_horizon = self.evict_horizon
        t.cnt_stride, t.sum_stride, t.sum_cstride = 1, 1, self.capacity
        t.cold_stride = t.hsum_stride = COLD_WORDS
        return t

    # -- accumulation ---------------------------------------------------------

    def accumulate_batch(self, index, fingerprint, contributions, frame: int | None = None,
                         ordered: bool | None = None, check: bool = True):
        """Insert a batch; returns (status u8, slot i64, probe_len u8) device tensors
        (src/table.py:117-142).  Raises ValueError on negative / non-finite input;
        check=False skips that pass (and its host sync) for inputs known to be valid."""
        if frame is None:
            frame = self.frame
        vals = as_f64(contributions, 3)
        if check:
            from .pipeline import check_contributions
            check_contributions(vals, torch.zeros(1, dtype=torch.int32, device=vals.device))
        idx = as_i64(index).reshape(-1)
        fp = as_u32_bits(fingerprint).reshape(-1)
        n = int(idx.shape[0])
        dev = idx.device
        status = torch.empty(n, dtype=torch.uint8, device=dev)
        slots = torch.empty(n, dtype=torch.int64, device=dev)
        probe_len = torch.empty(n, dtype=torch.uint8, device=dev)
        vtags = torch.empty(n, dtype=torch.int64, device=dev)
        vtouch = torch.empty(n, dtype=torch.int64, device=dev)
        use_ordered = self.ordered if ordered is None else bool(ordered)
        _lib.call("pf_accumulate_table", ctypes.byref(self.c_table()), idx.data_ptr(),
                  fp.data_ptr(), vals.data_ptr(), n, int(frame), int(use_ordered),
                  status.data_ptr(), slots.data_ptr(), probe_len.data_ptr(), vtags.data_ptr(),
                  vtouch.data_ptr(), _lib.stream_handle())
        self._pending_events.append((int(frame), status, slots, vtags, vtouch))
        return status, slots, probe_len

    def accumulate(self, h: CellHashes, contribution, frame: int | None = None,
                   key=None) -> InsertOutcome:
        """Single-vertex insert (spec-level API, src/table.py:144-156)."""
        status, slots, _ = self.accumulate_batch(
            np.array([h.index], np.uint64), np.array([h.fingerprint], np.uint32),
            np.asarray(contribution, np.float64).reshape(1, 3), frame)
        out = InsertOutcome(Outcome(int(status[0])), int(slots[0]))
        if self.shadow is not None and out.status is not Outcome.PROBE_LIMIT_EXCEEDED:
            if out.status is Outcome.EVICTED_THEN_ACCUMULATED:
                self.shadow[out.slot] = set()
            if key is not None:
                self.shadow.setdefault(out.slot, set()).add(key)
        return out

    @property
    def eviction_events(self) -> list[EvictionEvent]:
        """Eviction log (src/table.py:137-141); synchronises pending device results."""
        while self._pending_events:
            self._drain_front()
        return self._events

    def _drain_front(self):
        frame, status, slots, vtags, vtouch = self._pending_events.pop(0)
        if callable(status):  # a fused-frame log (producer closure, see pipeline.py)
            self._events.extend(status())
            return
        st = status.cpu().numpy()
        ev = np.nonzero(st == 1)[0]
        if len(ev):
            sl = slots.cpu().numpy()
            vt = u64_numpy(vtags)
            vtt = vtouch.cpu().numpy()
            for i in ev:
                age = (int(vt[i]) >> 32) & _AGE_MASK
                self._events.append(EvictionEvent(frame, int(sl[i]), age, int(vtt[i])))

    def _add_pending_events(self, producer, tag=None):
        self._pending_events.append((tag, producer, None, None, None))

    def _drain_tag(self, tag):
        """Drain, in order, every pending log up to and including the last one with `tag`
        (its device buffer is about to be reused); later logs stay pending."""
        idx = [k for k, p in enumerate(self._pending_events) if callable(p[1]) and p[0] == tag]
        for _ in range(idx[-1] + 1 if idx else 0):
            self._drain_front()

    # -- queries --------------------------------------------------------------

    def lookup_slots(self, index, fingerprint) -> torch.Tensor:
        idx = as_i64(index).reshape(-1)
        fp = as_u32_bits(fingerprint).reshape(-1)
        out = torch.empty(idx.shape[0], dtype=torch.int64, device=idx.device)
        _lib.call("pf_lookup_slots", self.tags.data_ptr(), self.capacity, idx.data_ptr(),
                  fp.data_ptr(), int(idx.shape[0]), self.probe_limit, out.data_ptr(),
                  _lib.stream_handle())
        return out

    def mean_at(self, slots, sums=None, counts=None) -> torch.Tensor:
        """Per-slot mean radiance (src/table.py:166-174); slots valid with count > 0."""
        sums = self.sums if sums is None else sums
        counts = self.counts if counts is None else counts
        s = as_i64(slots).reshape(-1)
        c = counts[s].to(torch.float64)
        if self.sum_mode == "fixed" and sums.dtype == torch.int64:
            return sums[s].to(torch.float64) / (c * FIXED_SCALE)[:, None]
        return sums[s] / c[:, None]

    def lookup(self, h: CellHashes):
        """(mean, count) of the live generation, or None when absent (src/table.py:176-184)."""
        slots = self.lookup_slots(np.array([h.index], np.uint64), np.array([h.fingerprint], np.uint32))
        s = int(slots[0])
        if s < 0 or int(self.counts[s]) == 0:
            return None
        mean = self.mean_at(np.array([s]))[0].cpu().numpy()
        return mean, int(self.counts[s])

    def probe_scan(self, h: CellHashes, accept) -> list:
        """All occupied window slots whose fingerprint satisfies `accept` (src/table.py:186-203).
        The window's tags and counts come back in one gather; `accept` is the caller's
        Python predicate, so the filter runs on the host; the accepted slots' means are one
        device call."""
        mask = self.capacity - 1
        home = int(h.index) & mask
        window = [(home + j) & mask for j in range(self.probe_limit)]
        w = torch.tensor(window, dtype=torch.int64, device=self.tags.device)
        tags = u64_numpy(self.tags[w])
        cnts = self.counts[w].cpu().numpy()
        hits = [j for j in range(len(window))
                if (int(tags[j]) & 0xFFFFFFFF) != 0 and cnts[j] != 0
                and accept(int(tags[j]) & 0xFFFFFFFF)]
        if not hits:
            return []
        means = self.mean_at(np.array([window[j] for j in hits])).cpu().numpy()
        return [(means[k], int(cnts[j])) for k, j in enumerate(hits)]

    def effective(self, mode: str, ema_alpha: float = 0.8, delta_max: float = 0.5):
        """Temporally blended (sum, count) per slot (src/table.py:205-238)."""
        code = temporal_code(mode)
        dev = self.tags.device
        as_int = code == 0 and self.sum_mode == "fixed"
        es = torch.empty((self.capacity, 3), dtype=torch.int64 if as_int else torch.float64,
                         device=dev)
        ec = torch.empty(self.capacity, dtype=torch.int64 if code == 0 else torch.float64,
                         device=dev)
        t = self.c_table()
        _lib.call("pf_effective", ctypes.byref(t), code, float(ema_alpha), float(delta_max),
                  es.data_ptr(), ec.data_ptr(), _lib.stream_handle())
        return es, ec

    # -- frame maintenance ----------------------------------------------------

    def begin_frame(self, frame: int, cfg: FilterConfig | None = None):
        """Fold live into history, re-prioritise, clear stale cells (src/table.py:242-298)."""
        mode = cfg.temporal_mode if cfg else "integrate"
        ema = cfg.ema_alpha if cfg else 0.8
        dmax = cfg.delta_max if cfg else 0.5
        cap = cfg.sample_cap if cfg else 0
        t = self.c_table()
        if self.shadow is not None:
            before = self.tags.clone()
        _lib.call("pf_begin_frame", ctypes.byref(t), int(frame), temporal_code(mode), float(ema),
                  float(dmax), int(cap), self._clears.data_ptr(), _lib.stream_handle())
        if self.shadow is not None:
            cleared = torch.nonzero((before != EMPTY_TAG_I64) & (self.tags == EMPTY_TAG_I64))
            for s in cleared.reshape(-1).cpu().numpy():
                self.shadow.pop(int(s), None)
        self.frame = frame

    @property
    def horizon_clears(self) -> int:
        return int(self._clears.item())

    # -- introspection --------------------------------------------------------

    def occupied_count(self) -> int:
        out = torch.zeros(1, dtype=torch.int64, device=self.tags.device)
        _lib.call("pf_count_occupied", self.tags.data_ptr(), self.capacity, out.data_ptr(),
                  _lib.stream_handle())
        return int(out.item())

    def occupancy(self) -> float:
        return self.occupied_count() / self.capacity

    def total_counts(self) -> int:
        return int(self.counts.sum().item())

    def total_sums(self) -> np.ndarray:
        return self.sums.sum(dim=0).cpu().numpy()

    def set_deltas(self, slots, values):
        s = as_i64(slots).reshape(-1)
        self.deltas[s] = as_f64(values).reshape(-1)

    def state(self) -> dict:
        """Host snapshot of every array with the reference dtypes."""
        return {"tags": u64_numpy(self.tags), "sums": self.sums.cpu().numpy(),
                "counts": self.counts.cpu().numpy(), "hist_sums": self.hist_sums.cpu().numpy(),
                "hist_counts": self.hist_counts.cpu().numpy(),
                "last_touch": self.last_touch.cpu().numpy(), "deltas": self.deltas.cpu().numpy()}

    def load_state(self, st: dict):
        """Replace the device state with host arrays (reference layout)."""
        self.tags.copy_(as_i64(st["tags"]))
        self.sums.copy_(torch.from_numpy(np.asarray(st["sums"])).to(self.sums))
        self.counts.copy_(as_i64(st["counts"]))
        self.hist_sums.copy_(torch.from_numpy(np.asarray(st["hist_sums"])).to(self.hist_sums))
        self.hist_counts.copy_(as_i64(st["hist_counts"]))
        self.last_touch.copy_(as_i64(st["last_touch"]))
        self.deltas.copy_(as_f64(st["deltas"]).reshape(-1))

    def export_csv(self, path):
        """slot,fingerprint,count,sum_r,sum_g,sum_b for occupied slots (src/table.py:314-324)."""
        st = self.state()
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("slot,fingerprint,count,sum_r,sum_g,sum_b\n")
            for s in np.nonzero(st["tags"] != np.uint64(EMPTY_TAG))[0]:
                fp = int(st["tags"][s]) & 0xFFFFFFFF
                if self.sum_mode == "fixed":
                    r, g, b = (float(v) for v in fixed_to_float(st["sums"][s]))
                else:
                    r, g, b = (float(v) for v in st["sums"][s])
                fh.write(f"{int(s)},{fp},{int(st['counts'][s])},{r!r},{g!r},{b!r}\n")

    def dump(self, path):
        """Binary snapshot, byte-identical layout to src/table.py:326-334."""
        st = self.state()
        mode = 0 if self.sum_mode == "fixed" else 1
        with open(path, "wb") as fh:
            fh.write(_DUMP_MAGIC)
            fh.write(struct.pack("<QBQ", self.capacity, mode, self.frame))
            for k in ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch"):
                fh.write(np.ascontiguousarray(st[k]).tobytes())

    def audit_no_false_merge(self) -> int:
        if self.shadow is None:
            raise RuntimeError("shadow map not enabled")
        return sum(1 for ks in self.shadow.values() if len(ks) > 1)
