"""Drop-in kernel module for the reference backend switch (src/_backend.py:14-42).

Exposes exactly the contract of `pathfilter._native` (src/_native.pyx:261-295):
`NAME`, `accumulate_fixed`, `accumulate_float`, `lookup_slots`.  Table arrays are
mutated in place and fresh per-vertex arrays are returned.

* CUDA tensors: zero-copy, stream-ordered, results stay on the device.
* numpy arrays (what the reference VoxelTable passes): each host table gets a
  persistent device mirror (one per table, keyed by its tags buffer).  The host
  buffers are page-locked in place once (cudaHostRegister, released when numpy frees
  them), so staging runs at DMA rate.  Per call:
  - the arrays the insert reads (tags, sums, counts, last_touch) are uploaded -- the
    host stays authoritative, so host-side mutations between calls (begin_frame,
    set_deltas, ...) are always seen;
  - the sm_100a insert runs;
  - only the slots the batch wrote are copied back.  Every net write of the insert
    lands on some vertex's returned slot; an eviction (status 1) also zeroes that slot's
    history and delta.
  The whole sequence holds the table's lock, so concurrent calls from several threads
  on one table serialise: each call is one atomic batch, and the final table is a valid
  linearisation.  The reference promises the same for disjoint batches
  (src/table.py:121-123).
* Insert order: batches below 4096 vertices run the sequential-order kernel, so slot
  layouts equal the reference's threads=1 layout.  The reference itself only splits
  larger batches across threads (src/pipeline.py:138-149).  Larger batches run the
  parallel kernel: one valid concurrent order, as the reference's threaded native
  kernel gives.  PF_DROPIN_ORDER=sequential|parallel overrides this.

`intersect_closest` / `intersect_any` belong to the tracer, which is outside the
filter hot path; they raise NotImplementedError.
"""

from __future__ import annotations

import os
import threading
import weakref

import numpy as np
import torch

from . import _lib
from .keys import as_f64, as_i64, as_u32_bits

NAME = "b200"

_TABLE = ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas")
_READ = ("tags", "sums", "counts", "last_touch")   # what the insert reads
SEQUENTIAL_BELOW = 4096                             # src/pipeline.py:138 (threads split)

_registry_lock = threading.Lock()
_mirrors: dict = {}


def _host_view(a, name):
    a = np.asarray(a)
    if not a.flags.c_contiguous:
        raise ValueError(f"{name} must be C-contiguous")
    return a


_registered: set = set()
REGISTER_MIN_BYTES = 1 << 20   # small arrays may share pages; their copies are cheap anyway


def _unregister(ptr: int) -> None:
    _registered.discard(ptr)
    try:
        _lib.lib().pf_host_unregister(ptr)
    except Exception:  # noqa: BLE001 -- interpreter shutdown
        pass


def _register(a: np.ndarray) -> None:
    """Page-lock a large numpy buffer in place for DMA (pf_host_register); released
    when numpy frees the buffer's owner."""
    ptr = a.ctypes.data
    if a.nbytes < REGISTER_MIN_BYTES or ptr in _registered:
        return
    owner = a
    while isinstance(owner.base, np.ndarray):
        owner = owner.base
    if _lib.lib().pf_host_register(ptr, a.nbytes) != 0:
        return   # stays pageable: correct, only slower
    _registered.add(ptr)
    weakref.finalize(owner, _unregister, ptr)


class _Mirror:
    """Device copy of one host VoxelTable's seven arrays."""

    def __init__(self, tags: np.ndarray):
        self.lock = threading.Lock()
        self.capacity = int(tags.shape[0])
        self.host: dict = {}       # name -> (weakref to the host array, data pointer)
        self.dev: dict = {}

    def bind(self, name: str, a: np.ndarray) -> torch.Tensor:
        """The device buffer for host array `a` (re-registered if the host array changed)."""
        ref = self.host.get(name)
        if ref is None or ref[0]() is not a or ref[1] != a.ctypes.data:
            _register(a)
            self.host[name] = (weakref.ref(a), a.ctypes.data)
            dt = {np.dtype(np.uint64): torch.int64, np.dtype(np.int64): torch.int64,
                  np.dtype(np.float64): torch.float64}.get(a.dtype)
            if dt is None:
                raise ValueError(f"{name} has dtype {a.dtype}; the kernels take 64-bit arrays")
            self.dev[name] = torch.empty(a.shape, dtype=dt, device=_lib.require_cuda())
        return self.dev[name]

    def upload(self, name: str, a: np.ndarray) -> torch.Tensor:
        d = self.bind(name, a)
        d.copy_(torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a))
        return d


def _mirror(tags: np.ndarray) -> _Mirror:
    key = (tags.ctypes.data, int(tags.shape[0]))
    with _registry_lock:
        m = _mirrors.get(key)
        if m is None or (m.host.get("tags") and m.host["tags"][0]() is not tags):
            m = _Mirror(tags)
            _mirrors[key] = m
            weakref.finalize(tags, _mirrors.pop, key, None)
        return m


def _order(n: int) -> int:
    """1 = sequential-order kernel, 0 = parallel."""
    mode = os.environ.get("PF_DROPIN_ORDER", "auto")
    if mode == "sequential":
        return 1
    if mode == "parallel":
        return 0
    if mode != "auto":
        raise ValueError("PF_DROPIN_ORDER must be auto|sequential|parallel")
    return 1 if n < SEQUENTIAL_BELOW else 0


def _check_sum_dtype(arrays: dict, fixed: bool):
    want = np.int64 if fixed else np.float64
    for k in ("sums", "hist_sums"):
        a = arrays[k]
        dt = a.dtype if not isinstance(a, torch.Tensor) else \
            (np.int64 if a.dtype == torch.int64 else np.float64)
        if dt != want:
            raise ValueError(f"{k} must be {np.dtype(want).name} for this kernel")


def _launch(fixed, t: dict, capacity, i, f, v, n, frame, probe_limit, evict_min_age, ordered):
    dev = i.device
    status = torch.zeros(n, dtype=torch.uint8, device=dev)
    slots = torch.full((n,), -1, dtype=torch.int64, device=dev)
    probe_len = torch.zeros(n, dtype=torch.uint8, device=dev)
    vtags = torch.zeros(n, dtype=torch.int64, device=dev)
    vtouch = torch.zeros(n, dtype=torch.int64, device=dev)
    fn = "pf_accumulate_fixed" if fixed else "pf_accumulate_float"
    _lib.call(fn, *(t[k].data_ptr() for k in _TABLE), int(capacity),
              i.data_ptr(), f.data_ptr(), v.data_ptr(), n, int(frame), int(probe_limit),
              int(evict_min_age), int(ordered), status.data_ptr(), slots.data_ptr(),
              probe_len.data_ptr(), vtags.data_ptr(), vtouch.data_ptr(), _lib.stream_handle())
    return status, slots, probe_len, vtags, vtouch


def _to_host(t: torch.Tensor) -> np.ndarray:
    """Stream-ordered D2H into page-locked memory (the caller synchronises); the numpy
    result keeps the pinned buffer alive."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h.numpy()


def _accumulate(fixed: bool, tags, sums, counts, hist_sums, hist_counts, last_touch, deltas,
                idx, fp, vals, frame, probe_limit, evict_min_age):
    arrays = dict(zip(_TABLE, (tags, sums, counts, hist_sums, hist_counts, last_touch, deltas)))
    _check_sum_dtype(arrays, fixed)
    if isinstance(tags, torch.Tensor):   # device table: zero-copy
        i = as_i64(idx).reshape(-1)
        f = as_u32_bits(fp).reshape(-1)
        v = as_f64(vals, 3)
        n = int(i.shape[0])
        return _launch(fixed, arrays, tags.shape[0], i, f, v, n, frame, probe_limit,
                       evict_min_age, _order(n))
    host = {k: _host_view(a, k) for k, a in arrays.items()}
    cap = int(host["tags"].shape[0])
    for k, a in host.items():
        if a.shape[0] != cap:
            raise ValueError(f"{k} has {a.shape[0]} rows, tags has {cap}")
    i = as_i64(np.ascontiguousarray(idx, np.uint64)).reshape(-1)
    f = as_u32_bits(np.ascontiguousarray(fp, np.uint32)).reshape(-1)
    v = as_f64(np.ascontiguousarray(vals, np.float64), 3)
    n = int(i.shape[0])
    m = _mirror(host["tags"])
    with m.lock:
        dev = {k: (m.upload(k, host[k]) if k in _READ else m.bind(k, host[k])) for k in _TABLE}
        status, slots, probe_len, vtags, vtouch = _launch(
            fixed, dev, cap, i, f, v, n, frame, probe_limit, evict_min_age, _order(n))
        # copy back the slots this batch wrote
        written = torch.unique(slots[slots >= 0])
        evicted = torch.unique(slots[status == 1]).cpu().numpy()
        w = written.cpu().numpy()
        for k in _READ:
            h = host[k].view(np.int64) if host[k].dtype == np.uint64 else host[k]
            h[w] = dev[k].index_select(0, written).cpu().numpy()
        if evicted.size:
            host["hist_sums"][evicted] = 0
            host["hist_counts"][evicted] = 0
            host["deltas"][evicted] = 0.0
        outs = [_to_host(x) for x in (status, slots, probe_len, vtags, vtouch)]
        torch.cuda.current_stream().synchronize()
    outs[3] = outs[3].view(np.uint64)
    return tuple(outs)


def accumulate_fixed(tags, sums, counts, hist_sums, hist_counts, last_touch, deltas, idx, fp,
                     vals, frame, probe_limit, evict_min_age):
    return _accumulate(True, tags, sums, counts, hist_sums, hist_counts, last_touch, deltas,
                       idx, fp, vals, frame, probe_limit, evict_min_age)


def accumulate_float(tags, sums, counts, hist_sums, hist_counts, last_touch, deltas, idx, fp,
                     vals, frame, probe_limit, evict_min_age):
    return _accumulate(False, tags, sums, counts, hist_sums, hist_counts, last_touch, deltas,
                       idx, fp, vals, frame, probe_limit, evict_min_age)


def lookup_slots(tags, idx, fp, probe_limit):
    host = not isinstance(tags, torch.Tensor)
    if host:
        tags = _host_view(tags, "tags")
        i = as_i64(np.ascontiguousarray(idx, np.uint64)).reshape(-1)
        f = as_u32_bits(np.ascontiguousarray(fp, np.uint32)).reshape(-1)
    else:
        i = as_i64(idx).reshape(-1)
        f = as_u32_bits(fp).reshape(-1)
    out = torch.empty(i.shape[0], dtype=torch.int64, device=i.device)

    def run(t):
        _lib.call("pf_lookup_slots", t.data_ptr(), int(t.shape[0]), i.data_ptr(), f.data_ptr(),
                  int(i.shape[0]), int(probe_limit), out.data_ptr(), _lib.stream_handle())

    if not host:
        run(tags)
        return out
    m = _mirror(tags)
    with m.lock:
        run(m.upload("tags", tags))
        return out.cpu().numpy()


def intersect_closest(*_a, **_k):
    raise NotImplementedError("ray casting is phase one (tracer), outside the filter hot path")


def intersect_any(*_a, **_k):
    raise NotImplementedError("ray casting is phase one (tracer), outside the filter hot path")
