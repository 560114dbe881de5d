"""SPEC criterion 3 (variance reduction, the paper's Fig. 1 analogue) and the jitter half
of criterion 8 on the device: builtin Cornell box, 1 spp filtered (render_frame: trace,
accumulate, resolve) and 1 spp unfiltered (the same trace's plain Monte Carlo image)
against a 1024-spp image from the same tracer with another seed; MSE in linear
radiance.  The filter must cut the MSE by >= 3x, and jitter on must not raise it by
more than 1.5x over jitter off.

usage: python tools/variance_reduction.py [--size 128] [--ref-spp 1024] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def mse(a, b) -> float:
    return float(((a - b) ** 2).mean())


def measure(size: int = 128, ref_spp: int = 1024, seed: int = 1) -> dict:
    import torch

    import paper_1902_05942_b200 as pf
    from paper_1902_05942_b200.tracer import TraceOptions, trace

    # pixel-centred rays: the path-space noise the filter acts on, without pixel-coverage
    # noise (the reference's own image-error fixture, pkg/tests/conftest.py:17-26)
    opt = TraceOptions(pixel_jitter=False)
    scene = pf.load_scene("cornell", size, size)
    ref = trace(scene, ref_spp, seed + 1000, opt).image
    out = {"scene": f"cornell {size}x{size}, pixel-centred rays", "reference_spp": ref_spp}
    for jitter in (True, False):
        cfg = pf.FilterConfig(capacity=1 << (2 * size * size - 1).bit_length(), jitter=jitter)
        frames = pf.run_sequence(scene, cfg, spp=1, seed=seed, frames=1, options=opt)
        r = frames[-1]
        key = "jitter_on" if jitter else "jitter_off"
        out[key] = {"mse_filtered": mse(r.filtered, ref), "mse_unfiltered": mse(r.unfiltered, ref)}
        out[key]["reduction"] = out[key]["mse_unfiltered"] / out[key]["mse_filtered"]
    out["jitter_on_over_off"] = out["jitter_on"]["mse_filtered"] / out["jitter_off"]["mse_filtered"]
    torch.cuda.synchronize()
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--ref-spp", type=int, default=1024)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    out = measure(args.size, args.ref_spp)
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
