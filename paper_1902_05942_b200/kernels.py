"""Drop-in kernel module for the reference backend switch (src/_backend.py:14-42).

Exposes exactly the contract of `pathfilter._native` (src/_native.pyx:261-295):
`NAME`, `accumulate_fixed`, `accumulate_float`, `lookup_slots`.  Table arrays are
mutated in place and fresh per-vertex arrays are returned.

* numpy arrays (what the reference VoxelTable passes): the table is staged into
  HBM, updated by the sm_100a kernel and copied back in place.  Inserts run in
  sequential (reference threads=1) order so slot layouts match bit for bit.
* CUDA tensors: zero-copy, stream-ordered, results stay on the device.

`intersect_closest` / `intersect_any` belong to the tracer, which is outside the
filter hot path; they raise NotImplementedError.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .keys import as_f64, as_i64, as_u32_bits

NAME = "b200"

_TABLE = ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas")


def _stage(arrays: dict):
    """CUDA views of the seven table arrays (uploads numpy inputs)."""
    dev = _lib.require_cuda()
    out = {}
    for k, a in arrays.items():
        if isinstance(a, torch.Tensor):
            out[k] = a
        else:
            a = np.asarray(a)
            if not a.flags.c_contiguous:
                raise ValueError(f"{k} must be C-contiguous")
            if a.dtype == np.uint64:
                a = a.view(np.int64)
            out[k] = torch.from_numpy(a).to(dev)
    return out


def _writeback(arrays: dict, staged: dict):
    for k, a in arrays.items():
        if not isinstance(a, torch.Tensor):
            host = staged[k].cpu().numpy()
            np.asarray(a).view(host.dtype)[...] = host


def _accumulate(fixed: bool, tags, sums, counts, hist_sums, hist_counts, last_touch, deltas,
                idx, fp, vals, frame, probe_limit, evict_min_age):
    arrays = dict(zip(_TABLE, (tags, sums, counts, hist_sums, hist_counts, last_touch, deltas)))
    want = np.int64 if fixed else np.float64
    for k in ("sums", "hist_sums"):
        a = arrays[k]
        dt = a.dtype if not isinstance(a, torch.Tensor) else \
            (np.int64 if a.dtype == torch.int64 else np.float64)
        if dt != want:
            raise ValueError(f"{k} must be {np.dtype(want).name} for this kernel")
    host = not isinstance(tags, torch.Tensor)
    st = _stage(arrays)
    i = as_i64(idx).reshape(-1)
    f = as_u32_bits(fp).reshape(-1)
    v = as_f64(vals, 3)
    n = int(i.shape[0])
    dev = i.device
    status = torch.zeros(n, dtype=torch.uint8, device=dev)
    slots = torch.full((n,), -1, dtype=torch.int64, device=dev)
    probe_len = torch.zeros(n, dtype=torch.uint8, device=dev)
    vtags = torch.zeros(n, dtype=torch.int64, device=dev)
    vtouch = torch.zeros(n, dtype=torch.int64, device=dev)
    fn = "pf_accumulate_fixed" if fixed else "pf_accumulate_float"
    _lib.call(fn, *(st[k].data_ptr() for k in _TABLE), int(st["tags"].shape[0]),
              i.data_ptr(), f.data_ptr(), v.data_ptr(), n, int(frame), int(probe_limit),
              int(evict_min_age), int(host), status.data_ptr(), slots.data_ptr(),
              probe_len.data_ptr(), vtags.data_ptr(), vtouch.data_ptr(), _lib.stream_handle())
    if not host:
        return status, slots, probe_len, vtags, vtouch
    _writeback(arrays, st)
    return (status.cpu().numpy(), slots.cpu().numpy(), probe_len.cpu().numpy(),
            vtags.cpu().numpy().view(np.uint64), vtouch.cpu().numpy())


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
    t = _stage({"tags": tags})["tags"]
    i = as_i64(idx).reshape(-1)
    f = as_u32_bits(fp).reshape(-1)
    out = torch.empty(i.shape[0], dtype=torch.int64, device=i.device)
    _lib.call("pf_lookup_slots", t.data_ptr(), int(t.shape[0]), i.data_ptr(), f.data_ptr(),
              int(i.shape[0]), int(probe_limit), out.data_ptr(), _lib.stream_handle())
    return out.cpu().numpy() if host else out


def intersect_closest(*_a, **_k):
    raise NotImplementedError("ray casting is phase one (tracer), outside the filter hot path")


def intersect_any(*_a, **_k):
    raise NotImplementedError("ray casting is phase one (tracer), outside the filter hot path")
