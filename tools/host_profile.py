"""cProfile of the host side of filter_frame on a small stream (where the frame is
host-bound): python tools/host_profile.py [width height]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_05942_b200 as pf  # noqa: E402
from paper_1902_05942_b200 import rng  # noqa: E402
from paper_1902_05942_b200.scene import closed_box  # noqa: E402
from paper_1902_05942_b200.streams import camera_footprint  # noqa: E402
from paper_1902_05942_b200.tracer import multi_bounce_stream  # noqa: E402

w, h = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (420, 238)
vs, base = multi_bounce_stream(closed_box(w, h), 1, 1, rr_start=9)
cfg = pf.FilterConfig(capacity=1 << (2 * len(vs) - 1).bit_length(), footprint_scale=camera_footprint(h))
state = pf.FrameState.from_config(cfg)
for f in range(5):
    pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, f))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for f in range(200):
    pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, 5 + f))
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(40)
st.sort_stats("tottime").print_stats(25)
