"""A small end-to-end case for compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py

A filtered frame of the golden 128x128 Cornell stream (fused frame and the ordered
phase-by-phase path), a 2-rank sharded frame, a trace of the benchmark scene and a
hybrid render sequence -- every kernel of the library on small inputs.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_1902_05942_b200 as pf
    from paper_1902_05942_b200 import sharded
    from paper_1902_05942_b200.render import run_sequence
    from paper_1902_05942_b200.scene import closed_box, load_scene
    from paper_1902_05942_b200.tracer import multi_bounce_stream
    from oracle.golden import golden_cfg, golden_stream, load_golden

    d = load_golden("frame_cornell128.npz")
    vs = golden_stream(d)
    cfg = pf.FilterConfig(**golden_cfg(d, "fixed_cfg"))
    for ordered in (False, True):
        st = pf.FrameState.from_config(cfg, ordered=ordered)
        for f in range(2):
            pf.filter_frame(vs, d["base"], cfg, st, 1, 1 + f)
    half = len(vs.pixel) // 2
    parts = [pf.VertexStream.from_any(type("S", (), {k: getattr(vs, k)[r] for k in (
        "position", "normal", "omega_r", "contribution", "throughput", "pixel", "sample",
        "layer_id", "camera_distance")})()) for r in (np.arange(half), np.arange(half, 2 * half))]
    states = [sharded.ShardedState(cfg, r, 2) for r in range(2)]
    for f in range(2):
        sharded.run_loopback([sharded.filter_frame_sharded(parts[r], d["base"], cfg, states[r], 1,
                                                           3 + f, composite="reduce")
                              for r in range(2)])
    stream, base = multi_bounce_stream(closed_box(32, 18), 4, 1)
    st = pf.FrameState.from_config(pf.FilterConfig(capacity=2048))
    pf.filter_frame(stream, base, pf.FilterConfig(capacity=2048), st, 1, 1)
    run_sequence(load_scene("shadow-sweep", 16, 16), pf.FilterConfig(
        capacity=1024, temporal_mode="hybrid", reevaluate_fraction=0.5), 1, 2, frames=3)
    run_sequence(load_scene("cornell-glossy", 12, 12), pf.FilterConfig(capacity=512), 2, 2,
                 frames=2)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
