"""Per-rank cost of the key-sharded frame, measured on ONE GPU.

G virtual ranks (run_loopback: collectives served in-process, ranks run one after
another on the same device, nothing waits on another rank's kernels) each render
the full 1080p 4-bounce stream of their own sample, exactly the bench's N-GPU
workload.  Reports the frame time of the fused single-GPU path, and for each G the
loopback frame time / G = the compute a rank does per frame (the all-to-all
transfer time over NVLink is not included; it is a few MB per rank per frame).

    python tools/shard_sim.py [--worlds 1,2,4,8] [--frames 5]
    python tools/shard_sim.py --band --width 3840 --height 2160   # configs[4]: strong scaling

--band: ONE frame split into G pixel-row bands (bench --workload uhd4-band): rank r
traces its rows, composites its band; per-rank compute = loopback time / G.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--frames", type=int, default=5)
    ap.add_argument("--repeat", type=int, default=3,
                    help="timed runs per point; the fastest is reported (the loopback's "
                         "host work between the ranks' kernels makes single runs noisy)")
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--stream", default="traced", choices=["traced", "synthetic"])
    ap.add_argument("--band", action="store_true", help="one frame in G row bands")
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_1902_05942_b200 as pf
    from paper_1902_05942_b200 import rng, sharded
    from paper_1902_05942_b200.streams import camera_footprint, closed_box_stream

    W, H = args.width, args.height
    cap = 1 << (2 * W * H - 1).bit_length()
    cfg = pf.FilterConfig(capacity=cap, footprint_scale=camera_footprint(H))
    base = closed_box_stream(W, H, 1, 1)[1]
    out = {"workload": (f"{W}x{H} 4 bounces, one frame in G row bands" if args.band else
                        f"{W}x{H} 4 bounces per rank ({args.stream})"), "capacity": cap}

    def timed(fn, frames):
        for f in range(2):
            fn(f)
        torch.cuda.synchronize()
        best = None
        for rep in range(max(1, args.repeat)):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            s.record()
            for f in range(frames):
                fn(10 + rep * frames + f)
            e.record()
            torch.cuda.synchronize()
            r = (s.elapsed_time(e) / frames, (time.perf_counter() - t0) * 1e3 / frames)
            best = r if best is None or r[0] < best[0] else best
        return best

    from paper_1902_05942_b200.scene import closed_box
    from paper_1902_05942_b200.tracer import multi_bounce_stream

    def rank_stream(r):
        if args.stream == "synthetic":
            s, _ = closed_box_stream(W, H, 4, 1 + r)
            s["sample"] = s["sample"] + 4 * r
            return pf.VertexStream(**s)
        return multi_bounce_stream(closed_box(W, H), 4, 1, sample_offset=4 * r)[0]

    from paper_1902_05942_b200.tracer import band_stream
    if args.band:
        vs0, base = multi_bounce_stream(closed_box(W, H), 4, 1)
    else:
        vs0 = rank_stream(0)
    st0 = pf.FrameState.from_config(cfg)
    ms, wall = timed(lambda f: pf.filter_frame(vs0, base, cfg, st0, 1, rng.frame_seed(1, f),
                                               want_means=False), args.frames)
    out["fused_single_ms"] = ms
    del st0
    del vs0
    for G in [int(x) for x in args.worlds.split(",")]:
        rows = H // G
        if args.band:
            bands = [band_stream(closed_box(W, H), 4, 1, r * rows, (r + 1) * rows) for r in range(G)]
            streams = [b[0] for b in bands]
            bases = [b[1] for b in bands]
        else:
            streams = [rank_stream(r) for r in range(G)]
        states = [sharded.ShardedState(cfg, r, G, agg_capacity=1 << 21) for r in range(G)]

        def frame(f):
            if args.band:
                gens = [sharded.filter_frame_sharded(
                    streams[r], bases[r], cfg, states[r], 1, rng.frame_seed(1, f),
                    pixel_base=r * rows * W, composite="band", want_means=False)
                    for r in range(G)]
            else:
                gens = [sharded.filter_frame_sharded(
                    streams[r], base, cfg, states[r], G, rng.frame_seed(1, f),
                    composite="reduce", want_means=False) for r in range(G)]
            sharded.run_loopback(gens)

        ms, wall = timed(frame, args.frames)
        out[f"world{G}"] = {"loopback_ms": ms, "per_rank_ms": ms / G, "wall_ms": wall,
                            "regrows": sum(s.regrows for s in states)}
        del states, streams
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
