"""Host enqueue cost of one bench frame vs its device time: is the frame loop host-bound?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1902_05942_b200 as pf  # noqa: E402
from paper_1902_05942_b200 import rng  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "hd4"
bench.W_PIX, bench.H_PIX, bench.BOUNCES, bench.TEMPORAL, _ = bench.WORKLOADS[w]
cfg = bench.make_config(pf)
stream, base = bench.make_stream("traced")
vs = pf.VertexStream(**stream)
state = pf.FrameState.from_config(cfg)
for f in range(5):
    pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, f), want_means=True)
torch.cuda.synchronize()
K = 30
use_marks = len(sys.argv) > 2 and sys.argv[2] == "marks"
marks = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(K)]
for m in marks:
    for ev in m:
        ev.record()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
t0 = time.perf_counter()
host = []
for f in range(K):
    t1 = time.perf_counter()
    pf.filter_frame(vs, base, cfg, state, 1, rng.frame_seed(1, 5 + f), want_means=True,
                    phase_events=marks[f] if use_marks else None)
    host.append(time.perf_counter() - t1)
t_enq = time.perf_counter() - t0
e.record()
torch.cuda.synchronize()
gpu = s.elapsed_time(e) / K
print(f"{w} marks={use_marks}: device {gpu:.3f} ms/frame; host enqueue mean {sum(host) / K * 1e3:.3f} ms, "
      f"max {max(host) * 1e3:.3f} ms, total {t_enq * 1e3:.1f} ms for {K} frames")
