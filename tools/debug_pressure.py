"""Debug: corridor frames on the fused parallel path; after each frame print evictions
whose victim tag age disagrees with frame - victim_last_touch, and the tables' ages."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_05942_b200 as pf  # noqa: E402
from paper_1902_05942_b200.pipeline import FrameState  # noqa: E402
from paper_1902_05942_b200.render import render_frame  # noqa: E402
from paper_1902_05942_b200.scene import corridor  # noqa: E402

EMPTY = np.uint64(0xFFFFFFFF00000000)
ordered = len(sys.argv) > 1 and sys.argv[1] == "ordered"
scene = corridor(48, 32, frames=40)
cfg = pf.FilterConfig(capacity=512, probe_limit=8, evict_min_age=3,
                      evict_horizon=8).for_camera(scene.camera.fov, scene.camera.height)
print("cfg min_age", cfg.evict_min_age)
state = FrameState.from_config(cfg, ordered=ordered)
prev_touch = None
for f in range(12):
    res = render_frame(scene, cfg, state, 1, 5)
    tags = state.fine.tags.cpu().numpy().view(np.uint64)
    touch = state.fine.last_touch.cpu().numpy()
    cnt = state.fine.counts.cpu().numpy()
    occ = tags != EMPTY
    age = (tags >> np.uint64(32)) & np.uint64(0xFFFFFF)
    ev = [e for e in state.fine.eviction_events if e.frame == f]
    bad = [e for e in ev if e.victim_age != f - e.victim_last_touch]
    print(f"frame {f}: n={len(res.trace_result.vertices)} occ={int(occ.sum())} live={int((cnt>0).sum())}"
          f" ev={len(ev)} bad={len(bad)} stale_touch={int(((cnt>0)&(touch!=f)).sum())}")
    for e in bad[:5]:
        pt = prev_touch[e.slot] if prev_touch is not None else None
        print("   ", e, "prev-frame last_touch", pt, "now tag age", int(age[e.slot]),
              "touch", int(touch[e.slot]), "cnt", int(cnt[e.slot]))
    prev_touch = touch.copy()
