"""Synthetic vertex buffers of the benchmark shape (BASELINE.json configs 2-5).

The reference's inputs come from its CPU path tracer (phase one, out of scope).
The benchmark instead synthesises a stream of the same shape and statistics on
the device: the closed Cornell box of SURVEY App. B (camera inside, so every
primary ray hits a diffuse wall), one vertex per bounce for `bounces` diffuse
bounces with cosine-weighted directions, path length as camera_distance, and
`sample = bounce - 1` so every vertex owns a distinct jitter draw (App. B).
Radiance values are synthetic (positive, heavy-tailed); they only feed sums.
"""

from __future__ import annotations

import math

import torch

BOX = 5.5
CAMERA = (2.75, 2.75, 0.6)
LOOK_AT = (2.75, 2.75, 5.5)
FOV = 1.2
# wall albedos (white, red at x=0, green at x=5.5), src/scene.py-style materials
_WHITE = (0.73, 0.73, 0.73)
_RED = (0.65, 0.05, 0.05)
_GREEN = (0.12, 0.45, 0.15)


def camera_footprint(height: int) -> float:
    """footprint_scale of FilterConfig.for_camera (src/keys.py:74-76) for this camera."""
    return 2.0 * math.tan(FOV / 2.0) / height


def _box_hit(o: torch.Tensor, d: torch.Tensor):
    """Exit point of rays starting inside [0, BOX]^3: (t, axis, side)."""
    inv = 1.0 / torch.where(d == 0, torch.full_like(d, 1e-300), d)
    t_far = torch.where(d > 0, (BOX - o) * inv, (0.0 - o) * inv)
    t_far = torch.where(d == 0, torch.full_like(t_far, float("inf")), t_far)
    t, axis = t_far.min(dim=1)
    side = (d.gather(1, axis[:, None])[:, 0] > 0)
    return t, axis, side


def closed_box_stream(width: int, height: int, bounces: int = 4, seed: int = 1,
                      device=None) -> tuple[dict, torch.Tensor]:
    """Vertex stream (dict of CUDA tensors with the reference field names) and a base image."""
    dev = torch.device(device) if device is not None else torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    npix = width * height
    pix = torch.arange(npix, device=dev, dtype=torch.int64)
    col = (pix % width).to(torch.float64)
    row = (pix // width).to(torch.float64)
    jx = torch.rand(npix, generator=g, device=dev, dtype=torch.float64)
    jy = torch.rand(npix, generator=g, device=dev, dtype=torch.float64)
    aspect = width / height
    th = math.tan(FOV / 2.0)
    sx = (2.0 * (col + jx) / width - 1.0) * th * aspect
    sy = (1.0 - 2.0 * (row + jy) / height) * th
    # camera looks down +z with +y up: right = forward x up = (-1, 0, 0)
    d = torch.stack([-sx, sy, torch.ones_like(sx)], dim=1)
    d = d / torch.linalg.norm(d, dim=1, keepdim=True)
    o = torch.tensor(CAMERA, device=dev, dtype=torch.float64).expand(npix, 3).clone()
    dist = torch.zeros(npix, device=dev, dtype=torch.float64)
    thr = torch.ones((npix, 3), device=dev, dtype=torch.float64)
    albedo = torch.tensor([_WHITE, _RED, _GREEN], device=dev, dtype=torch.float64)
    light = torch.tensor((2.75, 5.49, 2.75), device=dev, dtype=torch.float64)
    out = {k: [] for k in ("position", "normal", "omega_r", "contribution", "throughput",
                           "pixel", "sample", "layer_id", "camera_distance")}
    for k in range(bounces):
        t, axis, side = _box_hit(o, d)
        p = o + t[:, None] * d
        # snap the hit coordinate onto its wall exactly, as a plane intersection does
        wall = torch.where(side, torch.full_like(t, BOX), torch.zeros_like(t))
        p = p.scatter(1, axis[:, None], wall[:, None])
        n = torch.zeros_like(p).scatter(1, axis[:, None],
                                        torch.where(side, -1.0, 1.0).to(p.dtype)[:, None])
        dist = dist + t
        mat = torch.where((axis == 0) & ~side, 1, torch.where((axis == 0) & side, 2, 0))
        a = albedo[mat]
        ldist = torch.linalg.norm(p - light, dim=1)
        e = -torch.log1p(-torch.rand(npix, generator=g, device=dev, dtype=torch.float64))
        contrib = a * (0.9 / (0.5 + ldist * ldist) * e)[:, None]
        out["position"].append(p)
        out["normal"].append(n)
        out["omega_r"].append(-d)
        out["contribution"].append(contrib)
        out["throughput"].append(thr.clone())
        out["pixel"].append(pix)
        out["sample"].append(torch.full_like(pix, k))
        out["layer_id"].append(torch.zeros_like(pix))
        out["camera_distance"].append(dist.clone())
        if k + 1 == bounces:
            break
        # cosine-weighted bounce about the wall normal
        u1 = torch.rand(npix, generator=g, device=dev, dtype=torch.float64)
        u2 = torch.rand(npix, generator=g, device=dev, dtype=torch.float64)
        r = torch.sqrt(u1)
        ph = 2.0 * math.pi * u2
        lx, ly, lz = r * torch.cos(ph), r * torch.sin(ph), torch.sqrt(torch.clamp(1.0 - u1, min=0.0))
        loc = torch.stack([lx, ly, lz], dim=1)
        # axis-aligned frame: normal on `axis`, tangents on the other two axes
        perm = torch.stack([(axis + 1) % 3, (axis + 2) % 3, axis], dim=1)
        sign = torch.where(side, -1.0, 1.0).to(p.dtype)
        dn = torch.zeros_like(p)
        dn.scatter_(1, perm[:, 0:1], loc[:, 0:1])
        dn.scatter_(1, perm[:, 1:2], loc[:, 1:2])
        dn.scatter_(1, perm[:, 2:3], (loc[:, 2] * sign)[:, None])
        d = dn / torch.linalg.norm(dn, dim=1, keepdim=True)
        o = p + 1e-9 * n
        thr = thr * a
    stream = {k: torch.cat(v).contiguous() for k, v in out.items()}
    base = (0.05 * torch.rand((height, width, 3), generator=g, device=dev,
                              dtype=torch.float64)).contiguous()
    return stream, base


def stream_to_numpy(stream: dict):
    """Host copy with the reference field names (for the CPU baseline / oracle)."""
    class _S:
        pass
    s = _S()
    for k, v in stream.items():
        setattr(s, k, v.cpu().numpy())
    return s
