"""SPEC criterion 6 (constant-time scaling, paper §3.3.1) on the device: the per-vertex
time of one filtered frame (begin + accumulate + lookup, pf_filter_frame) across vertex
counts 1e5 .. 1e7 with proportional capacity (C = next_pow2(2 n), the CLI's default
rule).  Streams: the SURVEY App. B closed box, first hit (one vertex per pixel), at
resolutions giving each n.  Device time by CUDA events over K frames after W warm-up
frames (the frame is asynchronous: no host sync inside it).

usage: python tools/constant_time.py [--frames K] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (width, height): n = width * height first-hit vertices
SIZES = [(420, 238), (768, 432), (1332, 750), (2400, 1350), (4216, 2372)]


def measure(width: int, height: int, frames: int = 20, warmup: int = 3) -> dict:
    import torch

    import paper_1902_05942_b200 as pf
    from paper_1902_05942_b200 import rng
    from paper_1902_05942_b200.scene import closed_box
    from paper_1902_05942_b200.streams import camera_footprint
    from paper_1902_05942_b200.tracer import multi_bounce_stream

    vs, base = multi_bounce_stream(closed_box(width, height), 1, 1, rr_start=9)
    n = len(vs)
    cap = 1 << (2 * n - 1).bit_length()
    cfg = pf.FilterConfig(capacity=cap, footprint_scale=camera_footprint(height))
    state = pf.FrameState.from_config(cfg)
    for f in range(warmup):
        pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, f), want_means=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(frames):
        pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, warmup + f), want_means=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / frames
    # the frame's own device span: its first kernel's start to its last kernel's end
    # (phase events recorded inside the C call), without the host's per-call time
    marks = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(frames)]
    for m in marks:  # materialise (torch creates the event at its first record)
        for ev in m:
            ev.record()
    torch.cuda.synchronize()
    for f in range(frames):
        pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, warmup + frames + f),
                        want_means=True, phase_events=marks[f])
    torch.cuda.synchronize()
    dev_ms = sorted(m[0].elapsed_time(m[3]) for m in marks)[frames // 2]
    phases = {k: sorted(m[i].elapsed_time(m[i + 1]) for m in marks)[frames // 2]
              for i, k in enumerate(("begin_check", "insert", "resolve"))}
    del state
    torch.cuda.empty_cache()
    return {"width": width, "height": height, "vertices": n, "capacity": cap,
            "ms_per_frame": ms, "ns_per_vertex": ms * 1e6 / n,
            "device_ms_per_frame": dev_ms, "device_ns_per_vertex": dev_ms * 1e6 / n,
            "device_phases_ms": phases}


def sweep(frames: int = 20) -> dict:
    rows = [measure(w, h, frames) for w, h in SIZES]
    per = [r["ns_per_vertex"] for r in rows]
    dev = [r["device_ns_per_vertex"] for r in rows]
    return {"criterion": "SPEC 6: per-vertex accumulate+lookup time varies < 2x over 1e5..1e7",
            "rows": rows, "max_over_min": max(per) / min(per),
            "device_max_over_min": max(dev) / min(dev),
            "decades": math.log10(rows[-1]["vertices"] / rows[0]["vertices"])}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    out = sweep(args.frames)
    for r in out["rows"]:
        print(f"n={r['vertices']:>10,d} C=2^{r['capacity'].bit_length() - 1:<2d} "
              f"{r['ms_per_frame']:8.4f} ms/frame  {r['ns_per_vertex']:.4f} ns/vertex   "
              f"device {r['device_ms_per_frame']:8.4f} ms/frame "
              f"{r['device_ns_per_vertex']:.4f} ns/vertex  "
              + " ".join(f"{k} {v:.4f}" for k, v in r["device_phases_ms"].items()))
    print(f"max/min per-vertex time: {out['max_over_min']:.2f} (frame loop), "
          f"{out['device_max_over_min']:.2f} (device span)")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
