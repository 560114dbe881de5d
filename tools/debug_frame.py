"""Diagnose resolve mismatches against a golden fixture (GPU)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1902_05942_b200 as pf  # noqa: E402
from oracle.golden import golden_cfg, golden_stream, load_golden  # noqa: E402

fixture = sys.argv[1] if len(sys.argv) > 1 else "frame_box4.npz"
mode = sys.argv[2] if len(sys.argv) > 2 else "fixed"
d = load_golden(fixture)
vs = golden_stream(d)
cfg = pf.FilterConfig(**golden_cfg(d, f"{mode}_cfg"))
state = pf.FrameState.from_config(cfg)
seed = int(d["seed"])
image, report, stats = pf.filter_frame(vs, d["base"], cfg, state, 1, seed)
torch.cuda.synchronize()
src = report.source.cpu().numpy()
want = d[f"{mode}_source"]
bad = np.nonzero(src != want)[0]
print("mismatch rows", len(bad), "of", len(src), "mine", np.bincount(src, minlength=4),
      "gold", np.bincount(want, minlength=4))
work_n = int(state.scratch["work_count"].sum().item())
work = state.scratch["work"][:6 * work_n].view(-1, 6).cpu().numpy()
print("work rows", work_n, "fallback stat", int(report.counters[9].item()),
      "unique rows", len(np.unique(work[:, 0])))
lk = pf.vertex_keys(vs, cfg, seed, 3, 0).numpy()
ck = pf.vertex_keys(vs, cfg, seed, 3, cfg.coarse_delta).numpy()
es, ec = state.fine.effective(cfg.temporal_mode)
ces, cec = state.coarse.effective(cfg.temporal_mode)
ec = ec.cpu().numpy()
cec = cec.cpu().numpy()
for i in bad[:8]:
    inwork = np.nonzero(work[:, 0] == i)[0]
    rec = work[inwork[0]] if len(inwork) else None
    pool = 0
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                hi, hf = pf.hash_arrays([lk["qx"][i] + dx], [lk["qy"][i] + dy], [lk["qz"][i] + dz],
                                        [lk["level"][i]], lk["aux"][i:i + 1])
                s = int(state.fine.lookup_slots(hi, hf)[0])
                if s >= 0:
                    pool += ec[s]
    cs = int(state.coarse.lookup_slots(ck["index"][i:i + 1], ck["fingerprint"][i:i + 1])[0])
    ch = report.means[i].cpu().numpy()
    print(f"  work pos {inwork} chosen mine {ch} gold {d[f'{mode}_chosen'][i]} "
          f"contrib {vs.contribution[i]}")
    print(f"row {i}: mine {src[i]} gold {want[i]} in_work {len(inwork)} rec {rec} "
          f"key {(lk['qx'][i], lk['qy'][i], lk['qz'][i], lk['level'][i], lk['aux'][i])} "
          f"pool_cnt {pool} coarse_slot {cs} coarse_cnt {cec[cs] if cs >= 0 else None}")
import os
if os.environ.get("PF_DEBUG_RESOLVE"):
    work = state.scratch["work"][:6 * work_n].view(-1, 6).cpu().numpy()
    for i in bad[:8]:
        r = work[work[:, 0] == i][0]
        print("dbg row", i, "fm", hex(r[1]), "pic", r[2], "cnt_c", np.int64(r[3]).view(np.float64), "src*100+okc*10+anyn", r[4], "thr", np.int64(r[5]).view(np.float64))
