"""Frame time of back-to-back filter_frame calls with and without the input check /
the eviction-log read-back (what the per-frame host protocol costs on the stream).

    python tools/frame_gap.py
"""
import sys, time, torch
sys.path.insert(0, '.')
import __graft_entry__; __graft_entry__.build()
import paper_1902_05942_b200 as pf
from paper_1902_05942_b200 import rng, pipeline
from paper_1902_05942_b200.scene import closed_box
from paper_1902_05942_b200.tracer import multi_bounce_stream
from paper_1902_05942_b200.streams import camera_footprint
vs, base = multi_bounce_stream(closed_box(1920, 1080), 4, 1)
cfg = pf.FilterConfig(capacity=1 << 22, footprint_scale=camera_footprint(1080))
def run(label, **kw):
    st = pf.FrameState.from_config(cfg)
    for f in range(5): pf.filter_frame(vs, base, cfg, st, 1, rng.frame_seed(1, f), **kw)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for f in range(20): pf.filter_frame(vs, base, cfg, st, 1, rng.frame_seed(1, 10 + f), **kw)
    e.record(); torch.cuda.synchronize()
    print(label, s.elapsed_time(e) / 20)
run("default")
run("novalidate", validate=False)
orig = pipeline._register_event_drain
pipeline._register_event_drain = lambda *a, **k: None
run("nodrain")
run("nodrain_novalidate", validate=False)
pipeline._register_event_drain = orig
run("default2")
