"""Distinct fine / coarse keys per warp, per 256-vertex tile and per persistent CTA's
tile set on the bench stream: how much a CTA-level merge would save over the warp merge."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1902_05942_b200 as pf
from paper_1902_05942_b200 import rng

w = sys.argv[1] if len(sys.argv) > 1 else "hd4"
if w == "uhd4":
    bench.W_PIX, bench.H_PIX = 3840, 2160
stream, base = bench.make_stream("traced")
cfg = bench.make_config(pf)
vs = pf.VertexStream.from_any(type("S", (), stream)())
n = len(vs)
for name, delta in (("fine", 0), ("coarse", cfg.coarse_delta)):
    k = pf.vertex_keys(vs, cfg, 1, rng.STREAM_JITTER_ACCUM, delta)
    key = (k.index.to(torch.int64) & (cfg.capacity - 1)) | (k.fingerprint.to(torch.int64) << 32)
    total = torch.unique(key).numel()
    out = [f"{w} {name}: n={n} distinct={total}"]
    for group in (32, 256, 1024, 4096):
        m = (n // group) * group
        g = key[:m].view(-1, group)
        s, _ = torch.sort(g, dim=1)
        d = (s[:, 1:] != s[:, :-1]).sum().item() + g.shape[0]
        out.append(f"per{group}={d} ({m / d:.2f} v/upd)")
    print(" ".join(out), flush=True)
    # persistent CTAs: CTA c takes tiles c, c + G, ... (G = 148 SMs x 3 CTAs); distinct
    # keys per CTA over windows of `win` consecutive tiles of that CTA
    G, T = 444, 256
    ntile = n // T
    tiles = key[:ntile * T].view(ntile, T)
    res = []
    for win in (4, 16, 64, 10 ** 9):
        upd = 0
        for c in range(G):
            mine = tiles[c::G]
            for s0 in range(0, mine.shape[0], win):
                upd += torch.unique(mine[s0:s0 + win]).numel()
        res.append(f"cta_win{win if win < 10**9 else 'all'}={upd} ({ntile * T / upd:.2f} v/upd)")
    print(f"{w} {name}:", " ".join(res), flush=True)
