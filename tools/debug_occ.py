import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1902_05942_b200 as gpu
from paper_1902_05942_b200.pipeline import _occ_key
from oracle.golden import golden_cfg, golden_stream, load_golden
from oracle.digest import table_rows
d = load_golden("frame_cornell128.npz"); vs = golden_stream(d)
cfgd = golden_cfg(d, "fixed_cfg"); cfgd["capacity"] = 1 << 16; cfgd["evict_horizon"] = 3
cfg = gpu.FilterConfig(**cfgd)
A, B = gpu.FrameState.from_config(cfg), gpu.FrameState.from_config(cfg)
n = len(vs.pixel); rng = np.random.default_rng(3)
def rows(t):
    r = table_rows(t.state()); return {tuple(x[:1]): x for x in r} if False else r
for f in range(8):
    lo = (f * 1543) % (n // 2)
    sub = gpu.VertexStream.from_any(type("S", (), {k: getattr(vs, k)[lo:lo + n // 2] for k in ("position","normal","omega_r","contribution","throughput","pixel","sample","layer_id","camera_distance")})())
    B.scratch.pop("_occ_prev", None)
    if os.environ.get("BOTH_SWEEP"): A.scratch.pop("_occ_prev", None)
    prev = A.scratch.get("_occ_prev"); valid = prev is not None and prev[0] == _occ_key(A)
    if valid:
        i = prev[1]
        nf, nc = A.scratch[f"occ_n{i}"][:2].tolist()
        occf = A.scratch[f"occ_fine{i}"][:nf].cpu().numpy()
        truth = torch.nonzero(A.fine.tags != -(1 << 32)).flatten().cpu().numpy()
        print("frame", f, "list fine", nf, "occupied", len(truth), "same set", set(occf.tolist()) == set(truth.tolist()), "dups", nf - len(set(occf.tolist())))
        occc = A.scratch[f"occ_coarse{i}"][:nc].cpu().numpy()
        truthc = torch.nonzero(A.coarse.tags != -(1 << 32)).flatten().cpu().numpy()
        print("   list coarse", nc, "occupied", len(truthc), "same", set(occc.tolist()) == set(truthc.tolist()))
    ia, ra, _ = gpu.filter_frame(sub, d["base"], cfg, A, 1, 11 + f)
    ib, rb, _ = gpu.filter_frame(sub, d["base"], cfg, B, 1, 11 + f)
    print(f, "valid", valid, "img eq", np.array_equal(ia.cpu().numpy(), ib.cpu().numpy()),
          "src eq", np.array_equal(ra.source.cpu().numpy(), rb.source.cpu().numpy()))
    if f == 4:
        idx = rng.integers(0, 1 << 62, 64, dtype=np.int64).astype(np.uint64)
        fp = rng.integers(1, 1 << 32, 64, dtype=np.int64).astype(np.uint32)
        vals = rng.uniform(0, 1, (64, 3))
        for st in (A, B): st.fine.accumulate_batch(idx, fp, vals, f)
