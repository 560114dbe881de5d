"""Phase one on the device: trace paths and emit the vertex stream (src/tracer.py).

`trace` renders `spp` samples per pixel of a Scene with the sm_100a tracer kernel
(csrc/pf_trace.cu, one thread per path) and returns the plain Monte Carlo image,
the base image (radiance not routed through a recorded vertex) and the
VertexStream the filter consumes -- all CUDA tensors, so a frame goes from scene
to filtered image without touching the host.  `reevaluate` replays given path ids
(src/tracer.py:464-486).  Row order matches the reference's sequential trace:
samples in order, pixels in order within a sample.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .pipeline import VertexDescriptor, VertexStream  # noqa: F401  (src/tracer.py exports both)
from .scene import Scene

T_MIN = 1e-7
SHADOW_SHRINK = 1.0 - 1e-6


@dataclass
class TraceOptions:
    """src/tracer.py:35-43."""

    max_depth: int = 8
    rr_start: int = 3
    rr_clamp: tuple = (0.05, 0.95)
    nee: bool = True
    select_k: int = 1
    diffuse_threshold: float = 0.5
    pixel_jitter: bool = True

    def to_c(self) -> _lib.PfTraceOptions:
        o = _lib.PfTraceOptions()
        o.max_depth, o.rr_start, o.nee = int(self.max_depth), int(self.rr_start), int(self.nee)
        o.select_k, o.pixel_jitter = int(self.select_k), int(self.pixel_jitter)
        o.rr_lo, o.rr_hi = float(self.rr_clamp[0]), float(self.rr_clamp[1])
        o.diffuse_threshold = float(self.diffuse_threshold)
        return o


@dataclass
class TraceResult:
    """src/tracer.py:106-113 with device tensors."""

    image: torch.Tensor
    base_image: torch.Tensor
    vertices: VertexStream
    variance: torch.Tensor | None
    spp: int
    seed: int


def _device_scene(scene: Scene):
    """(PfScene, tensors) for a scene, cached on the scene object."""
    cache = scene.__dict__.get("_pf_device")
    if cache is not None and cache[0] is scene.v0 and cache[1] is scene.emission \
            and cache[2] is scene.camera:
        return cache[3], cache[4]
    _lib.require_cuda()
    tabs = scene.device_tables()
    cam = scene.camera
    right, up, fwd = cam.basis()
    tanf = math.tan(cam.fov / 2.0)
    aspect = cam.width / cam.height
    s = _lib.PfScene()
    for f in ("v0", "e1", "e2", "normal", "emission", "area", "material_id", "albedo",
              "glossy_weight", "glossy_exponent", "light_tri"):
        setattr(s, f, tabs[f].data_ptr())
    s.n_triangles = int(tabs["v0"].shape[0])
    s.n_materials = int(tabs["albedo"].shape[0])
    s.n_lights = int(tabs["light_tri"].shape[0])
    for name, vec in (("background", scene.background), ("cam_pos", cam.position),
                      ("cam_right", right), ("cam_up", up), ("cam_fwd", fwd)):
        getattr(s, name)[:] = [float(v) for v in vec]
    s.ndc_scale_x = 2.0 * tanf * aspect
    s.ndc_scale_y = 2.0 * tanf
    s.width, s.height = int(cam.width), int(cam.height)
    scene.__dict__["_pf_device"] = (scene.v0, scene.emission, scene.camera, s, tabs)
    return s, tabs


def trace_paths(scene: Scene, pixels: torch.Tensor, samples: torch.Tensor, seed: int,
                options: TraceOptions | None = None) -> dict:
    """Walk the given paths; per-path tensors (base, radiance, has_vertex, vertex fields)."""
    opt = options or TraceOptions()
    sc, keep = _device_scene(scene)
    dev = keep["v0"].device
    pixels = pixels.to(device=dev, dtype=torch.int64).contiguous()
    samples = samples.to(device=dev, dtype=torch.int64).contiguous()
    n = int(pixels.shape[0])
    out = {k: torch.empty((n, 3), dtype=torch.float64, device=dev)
           for k in ("base", "radiance", "position", "normal", "omega_r", "contribution",
                     "throughput")}
    out["has_vertex"] = torch.empty(n, dtype=torch.uint8, device=dev)
    out["layer_id"] = torch.empty(n, dtype=torch.int64, device=dev)
    out["camera_distance"] = torch.empty(n, dtype=torch.float64, device=dev)
    po = _lib.PfPathOut()
    for k, v in out.items():
        setattr(po, k, v.data_ptr())
    _lib.call("pf_trace_paths", ctypes.byref(sc), ctypes.byref(opt.to_c()),
              int(seed) & 0xFFFFFFFFFFFFFFFF, pixels.data_ptr(), samples.data_ptr(), n,
              ctypes.byref(po), _lib.stream_handle())
    out["pixel"], out["sample"] = pixels, samples
    return out


def _stream_of(paths: dict) -> VertexStream:
    rows = torch.nonzero(paths["has_vertex"]).reshape(-1)
    return VertexStream(position=paths["position"][rows], normal=paths["normal"][rows],
                        omega_r=paths["omega_r"][rows],
                        contribution=paths["contribution"][rows],
                        throughput=paths["throughput"][rows], pixel=paths["pixel"][rows],
                        sample=paths["sample"][rows], layer_id=paths["layer_id"][rows],
                        camera_distance=paths["camera_distance"][rows])


def concat_streams(streams: list) -> VertexStream:
    """VertexStream.concat (src/tracer.py:95-101)."""
    fields = ("position", "normal", "omega_r", "contribution", "throughput", "pixel", "sample",
              "layer_id", "camera_distance")
    return VertexStream.concat(streams)


def trace(scene: Scene, spp: int, seed: int, options: TraceOptions | None = None,
          threads: int = 1, sample_offset: int = 0, want_variance: bool = False,
          backend: str | None = None) -> TraceResult:
    """Render `spp` samples per pixel and collect the vertex stream (src/tracer.py:411-461).

    `threads` is accepted for signature compatibility: every pixel is one device thread,
    and the stream is always in the reference's threads=1 order (pixel-major per sample),
    which the reference documents as one valid ordering of the threads>1 stream."""
    _lib.check_backend(backend)
    if spp < 1:
        raise ValueError("spp must be >= 1")
    scene.validate()
    cam = scene.camera
    npix = cam.width * cam.height
    sc, keep = _device_scene(scene)
    dev = keep["v0"].device
    pix = torch.arange(npix, dtype=torch.int64, device=dev)
    total = torch.zeros((npix, 3), dtype=torch.float64, device=dev)
    base = torch.zeros_like(total)
    sq = torch.zeros_like(total) if want_variance else None
    streams = []
    for s in range(sample_offset, sample_offset + spp):
        paths = trace_paths(scene, pix, torch.full_like(pix, s), seed, options)
        total += paths["radiance"]
        base += paths["base"]
        if sq is not None:
            sq += paths["radiance"] ** 2
        streams.append(_stream_of(paths))
    var = None
    if want_variance:
        if spp > 1:
            var = torch.clamp((sq - total ** 2 / spp) / (spp - 1) / spp, min=0.0)
        else:
            var = torch.zeros_like(total)
        var = var.reshape(cam.height, cam.width, 3)
    return TraceResult((total / spp).reshape(cam.height, cam.width, 3),
                       (base / spp).reshape(cam.height, cam.width, 3),
                       streams[0] if len(streams) == 1 else concat_streams(streams), var, spp,
                       seed)


def reevaluate(scene: Scene, seed: int, spp: int, path_ids, options: TraceOptions | None = None,
               backend: str | None = None) -> VertexStream:
    """Replay paths by id under the current scene state (src/tracer.py:464-486)."""
    _lib.check_backend(backend)
    scene.validate()
    if isinstance(path_ids, torch.Tensor):
        ids = path_ids.to(torch.int64)
    else:
        ids = torch.as_tensor(np.asarray(path_ids, np.uint64).view(np.int64))
    npix = scene.camera.width * scene.camera.height
    pixels = ids & 0xFFFFFFFF
    samples = (ids >> 32) & 0xFFFFFFFF
    if len(ids) and (int(pixels.max()) >= npix or int(samples.max()) >= spp):
        raise ValueError("unknown path seed: pixel or sample index out of range")
    if len(ids) == 0:
        dev = _lib.require_cuda()
        e3 = torch.zeros((0, 3), dtype=torch.float64, device=dev)
        e1 = torch.zeros(0, dtype=torch.int64, device=dev)
        return VertexStream(e3, e3, e3, e3, e3, e1, e1, e1, e1.to(torch.float64))
    return _stream_of(trace_paths(scene, pixels, samples, seed, options))


def multi_bounce_stream(scene: Scene, bounces: int, seed: int, rr_start: int = 9,
                        options: TraceOptions | None = None, sample_offset: int = 0) -> tuple:
    """The benchmark stream of SURVEY App. B: select_k = 1..bounces traces at 1 spp,
    `sample += k - 1`, concatenated.  Returns (VertexStream, base image of k = 1).
    sample_offset traces another sample of every pixel (distinct path ids)."""
    streams, base = [], None
    for k in range(1, bounces + 1):
        opt = TraceOptions(**{**(options.__dict__ if options else {}), "select_k": k,
                              "rr_start": rr_start})
        res = trace(scene, 1, seed, opt, sample_offset=sample_offset)
        v = res.vertices
        v.sample = v.sample + (k - 1)
        streams.append(v)
        if base is None:
            base = res.base_image
    return concat_streams(streams), base


def band_stream(scene: Scene, bounces: int, seed: int, row_lo: int, row_hi: int,
                rr_start: int = 9, options: TraceOptions | None = None) -> tuple:
    """multi_bounce_stream restricted to the pixel rows [row_lo, row_hi): the stream of
    one rank of a frame split into pixel-row bands (the reference's thread split,
    src/pipeline.py:138-149 / src/tracer.py:429-434, across GPUs).  Concatenating the
    bands' streams in rank order gives, per select_k, the rows of the whole frame's
    stream.  Returns (VertexStream, base image rows [row_lo, row_hi) of k = 1)."""
    scene.validate()
    W = scene.camera.width
    _, keep = _device_scene(scene)
    dev = keep["v0"].device
    pix = torch.arange(row_lo * W, row_hi * W, dtype=torch.int64, device=dev)
    streams, base = [], None
    for k in range(1, bounces + 1):
        opt = TraceOptions(**{**(options.__dict__ if options else {}), "select_k": k,
                              "rr_start": rr_start})
        paths = trace_paths(scene, pix, torch.zeros_like(pix), seed, opt)
        v = _stream_of(paths)
        v.sample = v.sample + (k - 1)
        streams.append(v)
        if base is None:
            base = paths["base"].reshape(row_hi - row_lo, W, 3)
    return concat_streams(streams), base
