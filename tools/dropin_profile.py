"""Stage timings of the kernel-module drop-in's numpy path (one 10^6-vertex batch into
C = 2^22 tables), for tuning paper_1902_05942_b200/kernels.py."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
from pathfilter import _native, table  # noqa: E402

from paper_1902_05942_b200 import _lib, kernels  # noqa: E402

cap, n = 1 << 22, 1_000_000
r = np.random.default_rng(1)
keys = r.integers(0, 2**63, 60_000).astype(np.uint64)
b = table.VoxelTable(cap)
b._k = kernels
k = keys[:1000]
b.accumulate_batch(k, (k >> np.uint64(13)).astype(np.uint32) | np.uint32(1), np.ones((1000, 3)), 0)
print("registered", len(kernels._registered))
for rep in range(3):
    k = keys[r.integers(0, len(keys), n)]
    fp = (k >> np.uint64(13)).astype(np.uint32) | np.uint32(1)
    v = r.uniform(0, 4, (n, 3))
    torch.cuda.synchronize()
    T = {}
    t0 = time.perf_counter()
    vals = np.ascontiguousarray(v, np.float64)
    ok = np.any(~np.isfinite(vals)) or np.any(vals < 0.0)
    T["ref_checks"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    i = kernels.as_i64(np.ascontiguousarray(k, np.uint64))
    f = kernels.as_u32_bits(fp)
    vv = kernels.as_f64(vals, 3)
    torch.cuda.synchronize()
    T["inputs_h2d"] = time.perf_counter() - t0
    m = kernels._mirror(b.tags)
    host = {kk: getattr(b, kk) for kk in kernels._TABLE}
    t0 = time.perf_counter()
    dev = {kk: (m.upload(kk, host[kk]) if kk in kernels._READ else m.bind(kk, host[kk]))
           for kk in kernels._TABLE}
    torch.cuda.synchronize()
    T["table_h2d"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    out = kernels._launch(True, dev, cap, i, f, vv, n, 0, 32, 3, 0)
    torch.cuda.synchronize()
    T["kernel"] = time.perf_counter() - t0
    status, slots = out[0], out[1]
    t0 = time.perf_counter()
    written = torch.unique(slots[slots >= 0])
    w = written.cpu().numpy()
    torch.cuda.synchronize()
    T["unique"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for kk in kernels._READ:
        h = host[kk].view(np.int64) if host[kk].dtype == np.uint64 else host[kk]
        h[w] = dev[kk].index_select(0, written).cpu().numpy()
    T["writeback"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    o = [x.cpu().numpy() for x in out]
    T["outputs_d2h"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    b.accumulate_batch(k, fp, v, 0)
    T["whole_call"] = time.perf_counter() - t0
    print({kk: round(vv_ * 1e3, 2) for kk, vv_ in T.items()}, "written", len(w))
