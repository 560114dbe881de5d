"""Per-phase CUDA-event timings of the 1080p 4-bounce frame under config variants."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1902_05942_b200 as pf  # noqa: E402
from paper_1902_05942_b200 import rng  # noqa: E402
from paper_1902_05942_b200.streams import camera_footprint, closed_box_stream  # noqa: E402

W, H = 1920, 1080
stream, base = closed_box_stream(W, H, 4, 1)
vs = pf.VertexStream(**stream)
n = len(vs)


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(name, frames=6, **over):
    kw = dict(capacity=1 << 22, footprint_scale=camera_footprint(H))
    kw.update(over)
    cfg = pf.FilterConfig(**kw)
    st = pf.FrameState.from_config(cfg)
    acc = {"begin": 0.0, "insert": 0.0, "resolve": 0.0}
    for f in range(frames):
        seed = rng.frame_seed(1, f)
        e = [ev() for _ in range(6)]
        # each phase is enqueued behind a GPU sleep so the events bracket GPU time only
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e[0].record()
        st.fine.begin_frame(f, cfg)
        if st.coarse is not None:
            st.coarse.begin_frame(f, cfg)
        e[1].record()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e[4].record()
        fk, _, stats = pf.accumulate_phase(vs, cfg, st, f, seed, validate=False)
        e[2].record()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e[5].record()
        _, rep = pf.resolve_phase(vs, cfg, st, f, seed, 1, base, fk, want_means=False)
        e[3].record()
        torch.cuda.synchronize()
        if f >= 2:
            acc["begin"] += e[0].elapsed_time(e[1])
            acc["insert"] += e[4].elapsed_time(e[2])
            acc["resolve"] += e[5].elapsed_time(e[3])
    k = frames - 2
    occ = st.fine.occupied_count()
    cocc = st.coarse.occupied_count() if st.coarse is not None else 0
    fb = int(rep.counters[pf._lib.STAT_FALLBACK_ROWS].item()) if hasattr(rep, "counters") else -1
    print(f"{name:28s} begin {acc['begin']/k:7.3f} ms  insert {acc['insert']/k:7.3f} ms  "
          f"resolve {acc['resolve']/k:7.3f} ms  fine_occ {occ} coarse_occ {cocc} "
          f"fallback_rows {fb} probe_hist {dict(list(stats.probe_histogram.items())[:4])}")


def keys_only():
    cfg = pf.FilterConfig(capacity=1 << 22, footprint_scale=camera_footprint(H))
    for _ in range(2):
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        pf.vertex_keys(vs, cfg, 7, 2, 0)
        b.record()
        torch.cuda.synchronize()
    print(f"{'vertex_keys (1 key set)':28s} {a.elapsed_time(b):7.3f} ms (writes 76+24 B/vertex)")


print("vertices", n)
keys_only()
run("default")
run("no coarse", multi_level=False)
run("float sums", sum_mode="float")
run("filter mode", temporal_mode="filter")
run("no jitter", jitter=False)
