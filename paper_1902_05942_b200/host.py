"""Frames from host buffers: the call a reference user makes with numpy / pinned arrays.

`filter_frame` takes device tensors, or uploads host arrays synchronously.
`HostFramePipeline` is the streaming form.  Frame f+1's host-to-device copy runs on a copy
stream while frame f's kernels and its image read-back run on the compute stream.  Device
staging is double-buffered and reused, and events order every hand-off:
- copy(f) waits until frame f-2 has finished with its staging slot;
- frame f's kernels wait for copy(f);
- the read-back of frame f's image follows its kernels on the compute stream.

The H2D and D2H engines work in opposite directions, so a steady-state frame costs
max(H2D bytes / PCIe, kernels + D2H).  For the benchmark frame that is the PCIe copy.
Results are identical to `filter_frame` on the same inputs; only the copy schedule
differs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .keys import FilterConfig, device
from .pipeline import FrameState, VertexStream, filter_frame

_VEC = ("position", "normal", "omega_r", "contribution", "throughput")
_ALL = ("position", "normal", "omega_r", "contribution", "throughput", "pixel", "sample",
        "layer_id", "camera_distance")


def _needed(cfg: FilterConfig) -> tuple:
    """The stream fields the frame's kernels read (omega_r / layer_id only when a key
    option uses them, as validate_vertices requires)."""
    f = ["position", "normal", "contribution", "throughput", "pixel", "sample",
         "camera_distance"]
    if cfg.include_incident_angle:
        f += ["omega_r", "layer_id"]
    elif cfg.include_layer:
        f += ["layer_id"]
    return tuple(f)


def _host_tensor(a, dtype) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    if t.device.type != "cpu":
        raise ValueError("HostFramePipeline takes host arrays (numpy or CPU tensors)")
    return t.to(dtype).contiguous()


@dataclass
class HostFrame:
    """One submitted frame: `image` is a pinned host tensor, filled when `done` has fired
    and valid until the pipeline reuses its slot (`depth` submissions later)."""

    frame: int
    image: torch.Tensor
    report: object
    stats: object
    done: torch.cuda.Event

    def wait(self) -> torch.Tensor:
        self.done.synchronize()
        return self.image


class _Slot:
    def __init__(self):
        self.dev = {}
        self.base = None
        self.image = None
        self.free = None  # event: the frame that last used this slot has finished


class HostFramePipeline:
    """Stream frames from host memory through the filter with H2D/compute overlap."""

    def __init__(self, cfg: FilterConfig, state: FrameState | None = None, depth: int = 2):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.cfg = cfg
        self.state = state if state is not None else FrameState.from_config(cfg)
        self.dev = device()
        self.copy_stream = torch.cuda.Stream(device=self.dev)
        self.slots = [_Slot() for _ in range(depth)]
        self.count = 0
        self.fields = _needed(cfg)

    def _stage(self, slot: _Slot, name: str, shape, dtype) -> torch.Tensor:
        numel = int(np.prod(shape))
        buf = slot.dev.get(name)
        if buf is None or buf.numel() < numel:
            buf = torch.empty(max(numel, 1), dtype=dtype, device=self.dev)
            slot.dev[name] = buf
        return buf[:numel].view(shape)

    def submit(self, vertices, base_image, spp: int, seed: int, start_event=None) -> HostFrame:
        """Queue one frame.  `vertices` holds host arrays (pinned CPU tensors overlap; numpy
        or pageable tensors work but copy synchronously); `base_image` is (H, W, 3).
        `start_event` (optional) is a CUDA event the copies must wait for."""
        slot = self.slots[self.count % len(self.slots)]
        self.count += 1
        host = {}
        for f in self.fields:
            dt = torch.float64 if (f in _VEC or f == "camera_distance") else torch.int64
            host[f] = _host_tensor(getattr(vertices, f), dt)
        hbase = _host_tensor(base_image, torch.float64)
        n = int(host["pixel"].reshape(-1).shape[0])
        compute = torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(self.copy_stream):
            if start_event is not None:
                self.copy_stream.wait_event(start_event)
            if slot.free is not None:
                self.copy_stream.wait_event(slot.free)
            dev = {}
            for f in self.fields:
                d = self._stage(slot, f, host[f].shape, host[f].dtype)
                d.copy_(host[f], non_blocking=True)
                dev[f] = d
            dbase = self._stage(slot, "base", hbase.shape, hbase.dtype)
            dbase.copy_(hbase, non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(self.copy_stream)
        compute.wait_event(copied)
        for f in _ALL:  # fields no kernel reads this frame: empty placeholders
            if f not in dev:
                shape = (n, 3) if f in _VEC else (n,)
                dt = torch.float64 if (f in _VEC or f == "camera_distance") else torch.int64
                dev[f] = self._stage(slot, f, shape, dt)
        vs = VertexStream(**{f: dev[f] for f in _ALL})
        frame = self.state.frame
        image, report, stats = filter_frame(vs, dbase, self.cfg, self.state, spp, seed)
        if slot.image is None or slot.image.shape != image.shape:
            slot.image = torch.empty(image.shape, dtype=image.dtype).pin_memory()
        out = slot.image
        out.copy_(image, non_blocking=True)
        done = torch.cuda.Event()
        done.record(compute)
        slot.free = done
        return HostFrame(frame, out, report, stats, done)

    def run(self, frames) -> list:
        """Submit (vertices, base_image, spp, seed) tuples; return the host images in
        order.  A HostFrame's image buffer is reused `depth` frames later, so each image
        is copied out before its slot comes round again."""
        out, pending = [], []
        for f in frames:
            if len(pending) == len(self.slots):
                out.append(pending.pop(0).wait().clone())
            pending.append(self.submit(*f))
        return out + [p.wait().clone() for p in pending]
