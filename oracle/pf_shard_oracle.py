"""TEST INFRASTRUCTURE ONLY -- the owner-sliced table partition of SURVEY.md 8e, restated
over the sequential CPU oracle (oracle/pf_oracle.py).  Never imported by the product.

`ShardedTable` stands in for one global VoxelTable (src/table.py:80-340) of capacity C
but stores it as G owner slices: owner(home) = home >> (log2 C - log2 G), each owner a
plain oracle Table of capacity S = C/G addressed by home - owner*S, whose probe windows
wrap within the slice, so a probe chain never leaves its owner.  Feeding oracle.filter_frame a State of
ShardedTables shows on the reference's own fixtures that the partition the GPU ranks
use (paper_1902_05942_b200/sharded.py) leaves every per-key sum, count, source and
mean of src/pipeline.py:152-283 unchanged.

Slot ids seen by the pipeline are owner * S + local slot (the global slot when no
chain wraps).
"""

from __future__ import annotations

import numpy as np

from .pf_oracle import Table


class ShardedTable:
    def __init__(self, capacity, world, probe_limit=32, sum_mode="fixed", evict_horizon=8,
                 evict_min_age=3):
        if world < 1 or world & (world - 1) or capacity < world:
            raise ValueError("world must be a power of two <= capacity")
        self.capacity = capacity
        self.world = world
        self.slice = capacity // world
        self.local = self.slice
        self.shift = (capacity.bit_length() - 1) - (world.bit_length() - 1)
        self.sum_mode = sum_mode
        self.owners = [Table(self.local, probe_limit, sum_mode, evict_horizon, evict_min_age)
                       for _ in range(world)]

    @classmethod
    def from_config(cls, cfg, world: int) -> "ShardedTable":
        return cls(cfg.capacity, world, cfg.probe_limit, cfg.sum_mode, cfg.evict_horizon,
                   cfg.evict_min_age)

    def _route(self, index):
        home = np.asarray(index, np.uint64) & np.uint64(self.capacity - 1)
        owner = (home >> np.uint64(self.shift)).astype(np.int64)
        local = home - owner.astype(np.uint64) * np.uint64(self.slice)
        return owner, local

    def accumulate(self, index, fp, vals, frame):
        owner, local = self._route(index)
        fp = np.asarray(fp, np.uint32)
        vals = np.asarray(vals, np.float64)
        n = len(owner)
        st = np.zeros(n, np.uint8)
        sl = np.full(n, -1, np.int64)
        pl = np.zeros(n, np.uint8)
        vt = np.zeros(n, np.uint64)
        vtt = np.zeros(n, np.int64)
        for o, t in enumerate(self.owners):
            rows = np.nonzero(owner == o)[0]  # vertex order within the owner
            if len(rows) == 0:
                continue
            a, b, c, d, e = t.accumulate(local[rows], fp[rows], vals[rows], frame)
            st[rows], pl[rows], vt[rows], vtt[rows] = a, c, d, e
            sl[rows] = np.where(b >= 0, b + o * self.local, -1)
        return st, sl, pl, vt, vtt

    def lookup(self, index, fp):
        owner, local = self._route(index)
        fp = np.asarray(fp, np.uint32)
        out = np.full(len(owner), -1, np.int64)
        for o, t in enumerate(self.owners):
            rows = np.nonzero(owner == o)[0]
            if len(rows):
                s = t.lookup(local[rows], fp[rows])
                out[rows] = np.where(s >= 0, s + o * self.local, -1)
        return out

    def effective(self, mode, ema_alpha=0.8, delta_max=0.5):
        parts = [t.effective(mode, ema_alpha, delta_max) for t in self.owners]
        return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))

    def begin_frame(self, frame, cfg=None):
        for t in self.owners:
            t.begin_frame(frame, cfg)

    def cells(self) -> list:
        """Sorted (tag, count, hist_count, last_touch, sums, hist_sums) of occupied slots."""
        rows = []
        for t in self.owners:
            rows += table_cells(t)
        return sorted(rows)


def table_cells(t) -> list:
    occ = np.nonzero(t.tags != np.uint64(0xFFFFFFFF00000000))[0]
    return sorted((int(t.tags[s]), int(t.counts[s]), int(t.hist_counts[s]), int(t.last_touch[s]),
                   tuple(t.sums[s].tolist()), tuple(t.hist_sums[s].tolist())) for s in occ)
