"""Key-sharded multi-GPU filter frame.

One process per GPU.  The global fine and coarse tables (capacity C each, the
single-GPU layout) are split into G contiguous slices of home slots; rank r owns
homes [r*S, (r+1)*S), S = C/G, in a local table of capacity S whose probe windows wrap
within the slice (include/pathfilter_b200.h, section 3).

A frame is a generator that yields its collectives and receives their results:

    insert    keys of every local vertex; fine/coarse records pre-aggregated per
              distinct key and bucketed by owner              (pf_shard_keys / emit)
              -> all-to-all of counts (+ overflow / bad-input flags) and records
              owners apply the records                          (pf_shard_apply)
    publish   owners emit their occupied cells' effective records (pf_shard_publish)
              -> all-gather into a replica of the whole table   (pf_replica_update)
    resolve   every rank resolves its own vertices against the replica with the
              single-GPU rungs                                  (pf_resolve_replica)
    image     composite local to the rank's pixels ("band"), or summed over ranks with
              a reduce-scatter of the flat buffer ("reduce": ranks trace different
              samples of the same pixels), then base + flat / spp (pf_finalize_image)

`run_dist` drives a frame with torch.distributed (NCCL on B200; gloo copies through
host memory); `run_loopback` drives G virtual ranks in one process (tests).

Results equal the single-GPU frame over the ranks' concatenated vertex streams: each
key's records reach exactly one owner, 16.16 fixed-point sums are exactly associative,
and the replica holds the owners' cells verbatim, so every rung sees the same
effective (sum, count) values.  Only the slot a key occupies can differ (probe windows
wrap within a slice), which matters only when a chain reaches probe_limit.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, rng
from .keys import FilterConfig, as_f64, device, temporal_code
from .pipeline import FrameStats, ResolveReport, VertexStream
from .table import VoxelTable

_AGG_EMPTY = -1  # ~0 as int64
_EMPTY_TAG = 0xFFFFFFFF00000000 - (1 << 64)  # as int64


@dataclass
class Exchange:
    """One all-to-all: rows [sum(send_rows[:p]), +send_rows[p]) of `tensor` go to rank p;
    the result holds recv_rows[p] rows from each rank p, in rank order."""

    tensor: torch.Tensor
    send_rows: list
    recv_rows: list


@dataclass
class AllGather:
    """Concatenate every rank's `tensor` (same shape on all ranks) in rank order."""

    tensor: torch.Tensor


@dataclass
class ReduceScatter:
    """Sum `tensor` (rows divisible by world) over ranks; rank r receives block r."""

    tensor: torch.Tensor


def _next_pow2(x: int) -> int:
    return 1 << max(int(x) - 1, 1).bit_length()


class ShardedState:
    """This rank's slices of the fine/coarse tables, the aggregation scratch and the
    replica of the global tables used by the resolve."""

    def __init__(self, cfg: FilterConfig, rank: int, world: int, agg_capacity: int = 1 << 20):
        _lib.require_cuda()
        C = int(cfg.capacity)
        if world < 1 or world & (world - 1) or world > 64:
            raise ValueError("world must be a power of two <= 64")
        if C < 2 * world or C & (C - 1):
            raise ValueError("capacity must be a power of two >= 2 * world")
        if not 0 <= rank < world:
            raise ValueError("rank out of range")
        self.cfg_capacity = C
        self.rank, self.world = int(rank), int(world)
        self.slice = C // world
        self.fine = VoxelTable(self.slice, cfg.probe_limit, cfg.sum_mode, cfg.evict_horizon,
                               cfg.evict_min_age)
        self.coarse = (VoxelTable(self.slice, cfg.probe_limit, cfg.sum_mode, cfg.evict_horizon,
                                  cfg.evict_min_age) if cfg.multi_level else None)
        self.sum_mode = cfg.sum_mode
        self.probe_limit = int(cfg.probe_limit)
        self.frame = 0
        dev = device()
        self._dev = dev
        self.n_distinct = torch.zeros(1, dtype=torch.int64, device=dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.owner_counts = torch.zeros((2, world), dtype=torch.int64, device=dev)
        self.owner_cursor = torch.zeros((2, world), dtype=torch.int64, device=dev)
        self.bad_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self._alloc_agg(_next_pow2(max(int(agg_capacity), 64)))
        # replica of the global tables (tags EMPTY until published), published entries
        empty = torch.full((C,), _EMPTY_TAG, dtype=torch.int64, device=dev)
        self.rep_fine_tags = empty
        self.rep_fine_rec = torch.zeros((C, 4), dtype=torch.int64, device=dev)
        self.rep_coarse_tags = empty.clone() if self.coarse is not None else None
        self.rep_coarse_rec = (torch.zeros((C, 4), dtype=torch.int64, device=dev)
                               if self.coarse is not None else None)
        n_local = self.slice * (2 if self.coarse is not None else 1)
        self.entries = torch.empty((n_local, 6), dtype=torch.int64, device=dev)
        self.entry_count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.prev_gathered = None  # (entries [world * stride, 6], counts [world], stride)
        self.last_comm = None  # interconnect bytes of the last frame (filter_frame_sharded)
        # every rank's published entry count of the last frame, copied to pinned host
        # memory behind the frame's gather (read once the next frame's count exchange
        # has synchronised, i.e. after it has landed)
        self.prev_entry_counts = torch.zeros(world, dtype=torch.int64).pin_memory()
        self.scratch: dict = {}
        self.regrows = 0

    # -- buffers ------------------------------------------------------------------

    def _alloc_agg(self, cap: int):
        dev = self._dev
        self.agg_capacity = cap
        self.agg_keys = torch.full((cap,), _AGG_EMPTY, dtype=torch.int64, device=dev)
        self.agg_sums = torch.zeros((cap, 3), dtype=torch.int64, device=dev)
        self.agg_counts = torch.zeros(cap, dtype=torch.int64, device=dev)
        self.distinct = torch.empty(cap // 2, dtype=torch.int32, device=dev)
        self.send_records = torch.empty((cap // 2, 5), dtype=torch.int64, device=dev)
        self.send_requests = torch.empty(1, dtype=torch.int64, device=dev)

    def grow_agg(self, need: int):
        """Re-allocate the aggregation table for `need` distinct keys (empty)."""
        self._alloc_agg(_next_pow2(2 * int(need) + 2))
        self.n_distinct.zero_()
        self.overflow.zero_()
        self.owner_counts.zero_()
        self.regrows += 1

    def buffer(self, name: str, shape, dtype) -> torch.Tensor:
        n = int(np.prod(shape))
        b = self.scratch.get(name)
        if b is None or b.numel() < n or b.dtype != dtype:
            b = torch.empty(max(n, 1), dtype=dtype, device=self._dev)
            self.scratch[name] = b
        return b[:n].view(*shape)

    def c_shard(self) -> _lib.PfShard:
        s = _lib.PfShard()
        s.rank, s.world = self.rank, self.world
        s.log2_capacity = self.cfg_capacity.bit_length() - 1
        s.sum_mode = 0 if self.sum_mode == "fixed" else 1
        s.agg_keys, s.agg_sums = self.agg_keys.data_ptr(), self.agg_sums.data_ptr()
        s.agg_counts, s.agg_capacity = self.agg_counts.data_ptr(), self.agg_capacity
        s.distinct, s.n_distinct = self.distinct.data_ptr(), self.n_distinct.data_ptr()
        s.overflow = self.overflow.data_ptr()
        s.owner_counts, s.owner_cursor = self.owner_counts.data_ptr(), self.owner_cursor.data_ptr()
        return s

    def c_replica(self) -> _lib.PfReplica:
        r = _lib.PfReplica()
        r.fine_tags, r.fine_records = self.rep_fine_tags.data_ptr(), self.rep_fine_rec.data_ptr()
        r.coarse_tags = _lib.ptr(self.rep_coarse_tags)
        r.coarse_records = _lib.ptr(self.rep_coarse_rec)
        r.capacity = self.cfg_capacity
        r.slice_log2 = self.slice.bit_length() - 1
        r.probe_limit = self.probe_limit
        r.sum_mode = 0 if self.sum_mode == "fixed" else 1
        return r


def _stats_message(st: ShardedState) -> torch.Tensor:
    """[world, 3] int64 per destination: records, overflow, bad input (all-gathered: every
    rank sees the whole [world, world, 3] send matrix)."""
    cols = [st.owner_counts[0], st.overflow.to(torch.int64).expand(st.world),
            st.bad_flag.to(torch.int64).expand(st.world)]
    return torch.stack(cols, dim=1).contiguous()


def filter_frame_sharded(vertices, base_image, cfg: FilterConfig, st: ShardedState, spp: int,
                         seed: int, pixel_base: int = 0, composite: str = "band",
                         validate: bool = True, want_means: bool = True, phase_events=None):
    """One frame on this rank (generator: yields Exchange / AllGather / ReduceScatter).

    composite="band": the rank's vertices all land in its pixel band
    [pixel_base, pixel_base + H*W) and `base_image` is that band (H x W x 3).
    composite="reduce": every rank's vertices address the whole image of H x W
    pixels (pixel_base 0) -- e.g. each rank traced other samples -- and the result is
    this rank's block of rows of the final image (H divisible by world).
    phase_events: optional 4 torch.cuda.Events recorded at frame start, after the key
    kernel, after the replica is built and at frame end.

    Returns (image, ResolveReport, FrameStats) via StopIteration.value."""
    if composite not in ("band", "reduce"):
        raise ValueError("composite must be 'band' or 'reduce'")
    frame = st.frame
    vs = VertexStream.from_any(vertices)
    n = len(vs)
    base = as_f64(base_image)
    H, W = int(base.shape[0]), int(base.shape[1])
    G = st.world
    if composite == "reduce" and (H % G or pixel_base):
        raise ValueError("reduce composite needs H divisible by world and pixel_base 0")
    n_pix = H * W
    dev = base.device
    cc = cfg.to_c()
    v, keep = vs.c_struct()
    ft = st.fine.c_table()
    ct = st.coarse.c_table() if st.coarse is not None else None
    has_coarse = int(st.coarse is not None)
    stream = _lib.stream_handle()
    acc = torch.zeros(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
    res = torch.zeros(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
    accum_seed = rng.stream_base(seed, rng.STREAM_JITTER_ACCUM)
    lookup_seed = rng.stream_base(seed, rng.STREAM_JITTER_LOOKUP)
    coarse_seed = rng.stream_base(seed, rng.STREAM_JITTER_LOOKUP if cfg.jitter
                                  else rng.STREAM_JITTER_ACCUM)
    lk_keys = st.buffer("lk_keys", (max(n, 1),), torch.int64)  # packed fp << 32 | slot index

    def mark(k):
        if phase_events is not None:
            phase_events[k].record()

    mark(0)
    # temporal update on the local slices (src/pipeline.py:331-333) and the input check,
    # side by side in one launch
    check = validate and n > 0
    _lib.call("pf_begin_frame_checked", ctypes.byref(ft), ctypes.byref(ct) if ct is not None
              else None, int(frame), temporal_code(cfg.temporal_mode), float(cfg.ema_alpha),
              float(cfg.delta_max), int(cfg.sample_cap), st.fine._clears.data_ptr(),
              st.coarse._clears.data_ptr() if st.coarse is not None else None,
              vs.contribution.data_ptr() if check else None, 3 * n,
              st.bad_flag.data_ptr(), stream)
    st.fine.frame = frame
    if st.coarse is not None:
        st.coarse.frame = frame

    # ---- insert: pre-aggregated records to their owners.  The counts go by all-gather, so
    # every rank knows every rank's incoming record count: with last frame's entry counts
    # that bounds this frame's published entries, and the publish needs no second sync.
    while True:
        sh = st.c_shard()
        _lib.call("pf_shard_keys", ctypes.byref(cc), ctypes.byref(v), ctypes.byref(sh), has_coarse,
                  accum_seed, lookup_seed, st.bad_flag.data_ptr(), lk_keys.data_ptr(),
                  stream)
        mark(1)
        _lib.call("pf_shard_emit", ctypes.byref(sh), st.send_records.data_ptr(),
                  st.send_requests.data_ptr(), stream)
        msg = _stats_message(st)
        allm = (yield AllGather(msg)).reshape(G, G, 3).cpu().numpy()  # the frame's one sync
        if allm[:, :, 2].any():
            _lib.call("pf_shard_reset", ctypes.byref(sh), stream)
            raise ValueError("contributions must be finite and non-negative "
                             "(frame rejected on every rank; tables unchanged)")
        if not allm[:, 0, 1].any():
            break
        if allm[st.rank, 0, 1]:  # this rank overflowed: grow and redo its keys
            st.grow_agg(int(st.n_distinct.item()))
        else:  # a peer overflowed: keep this rank's round, repeat the count exchange
            st.overflow.zero_()
            msg = _stats_message(st)
            while True:
                allm = (yield AllGather(msg)).reshape(G, G, 3).cpu().numpy()
                if not allm[:, 0, 1].any():
                    break
            break
    send_rec = allm[st.rank, :, 0].tolist()
    recv_rec = allm[:, st.rank, 0].tolist()
    # this rank's interconnect bytes of the frame (what leaves / arrives over NVLink; the
    # self-addressed share of the all-to-all stays on the device)
    rec_b = st.send_records.element_size() * int(st.send_records[:1].numel())
    comm = {"count_allgather": msg.numel() * msg.element_size() * (G - 1),
            "records_sent": rec_b * (sum(send_rec) - send_rec[st.rank]),
            "records_received": rec_b * (sum(recv_rec) - recv_rec[st.rank])}
    # published entries of rank r <= its entries last frame + the records it receives
    bound = int((st.prev_entry_counts.numpy() + allm[:, :, 0].sum(axis=0)).max())
    records = yield Exchange(st.send_records[:sum(send_rec)], send_rec, recv_rec)
    _lib.call("pf_shard_apply", ctypes.byref(sh), ctypes.byref(ft),
              ctypes.byref(ct) if ct is not None else None, records.data_ptr(),
              int(records.shape[0]), int(frame), acc.data_ptr(), stream)
    _lib.call("pf_shard_reset", ctypes.byref(sh), stream)

    # ---- publish the owners' cells into every rank's replica
    _lib.call("pf_shard_publish", ctypes.byref(sh), ctypes.byref(cc), ctypes.byref(ft),
              ctypes.byref(ct) if ct is not None else None, st.entries.data_ptr(),
              st.entry_count.data_ptr(), stream)
    counts = yield AllGather(st.entry_count)
    stride = min(bound, int(st.entries.shape[0]))  # >= every rank's count; same on all ranks
    # every rank computed the same bound, so all skip an empty gather together
    gathered = (yield AllGather(st.entries[:stride])) if stride else st.entries[:0]
    ent_b = st.entries.element_size() * int(st.entries[:1].numel())
    comm["entries_allgather"] = ent_b * stride * (G - 1) + counts.element_size() * (G - 1)
    st.prev_entry_counts.copy_(counts, non_blocking=True)
    rp = st.c_replica()
    if st.prev_gathered is not None:
        pg, pc, ps = st.prev_gathered
        _lib.call("pf_replica_update", ctypes.byref(rp), pg.data_ptr(), pc.data_ptr(), G, ps, 1,
                  stream)
    counts_dev = counts.to(dev).contiguous()
    _lib.call("pf_replica_update", ctypes.byref(rp), _lib.ptr(gathered) if stride else None,
              counts_dev.data_ptr(), G, stride, 0, stream)
    st.prev_gathered = (gathered, counts_dev, stride)
    mark(2)

    # ---- resolve this rank's vertices against the replica
    source = torch.empty(n, dtype=torch.uint8, device=dev)
    chosen = torch.empty((n, 3), dtype=torch.float64, device=dev) if want_means else None
    flat = st.buffer("flat", (n_pix, 3), torch.float64)
    work = st.buffer("work", (_lib.work_rows(n),), torch.int64)
    work_count = st.buffer("work_count", (_lib.WORK_LISTS,), torch.int64)
    fb_keys = st.buffer("fallback_keys", (max(n, 1), 8), torch.int64)
    _lib.call("pf_resolve_replica", ctypes.byref(cc), ctypes.byref(v), ctypes.byref(rp),
              lookup_seed, coarse_seed, lk_keys.data_ptr(), flat.data_ptr(),
              n_pix, int(pixel_base), work.data_ptr(), work_count.data_ptr(), fb_keys.data_ptr(),
              source.data_ptr(), _lib.ptr(chosen), res.data_ptr(), stream)
    del keep

    # ---- image
    if composite == "reduce":
        band_flat = yield ReduceScatter(flat)
        rows = H // G
        base_band = base[st.rank * rows:(st.rank + 1) * rows]
        # ring reduce-scatter: (G - 1) / G of the buffer leaves each rank
        comm["image_reduce_scatter"] = flat.numel() * flat.element_size() * (G - 1) // G
    else:
        band_flat, base_band = flat, base
    image = torch.empty_like(base_band)
    _lib.call("pf_finalize_image", base_band.data_ptr(), band_flat.data_ptr(), image.data_ptr(),
              int(base_band.shape[0] * base_band.shape[1]), int(spp), stream)
    mark(3)
    st.last_comm = comm
    st.fine.frame = frame
    if st.coarse is not None:
        st.coarse.frame = frame
    st.frame = frame + 1
    report = ResolveReport(source, image, chosen)
    report.counters = res
    return image, report, FrameStats(frame=frame, n_vertices=n, counters=acc)


# ------------------------------------------------------------------ drivers

def _a2a_dist(ex: Exchange, group=None) -> torch.Tensor:
    import torch.distributed as dist
    t = ex.tensor.contiguous()
    out_shape = (int(sum(ex.recv_rows)),) + tuple(t.shape[1:])
    via_host = t.is_cuda and dist.get_backend(group) == "gloo"
    src = t.cpu() if via_host else t
    out = torch.empty(out_shape, dtype=t.dtype, device=src.device)
    dist.all_to_all_single(out, src, [int(x) for x in ex.recv_rows],
                           [int(x) for x in ex.send_rows], group=group)
    return out.to(t.device) if via_host else out


def _reduce_scatter_dist(rs: ReduceScatter, group=None) -> torch.Tensor:
    import torch.distributed as dist
    t = rs.tensor.contiguous()
    g = dist.get_world_size(group)
    rows = t.shape[0] // g
    via_host = t.is_cuda and dist.get_backend(group) == "gloo"
    src = t.cpu() if via_host else t
    if via_host:  # gloo has no reduce_scatter: all-reduce and keep this rank's block
        dist.all_reduce(src, group=group)
        r = dist.get_rank(group)
        return src[r * rows:(r + 1) * rows].to(t.device)
    out = torch.empty((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.reduce_scatter_tensor(out, src, group=group)
    return out


def _all_gather_dist(ag: AllGather, group=None) -> torch.Tensor:
    import torch.distributed as dist
    t = ag.tensor.contiguous()
    g = dist.get_world_size(group)
    via_host = t.is_cuda and dist.get_backend(group) == "gloo"
    src = t.cpu() if via_host else t
    if via_host:
        parts = [torch.empty_like(src) for _ in range(g)]
        dist.all_gather(parts, src, group=group)
        return torch.cat(parts).to(t.device)
    out = torch.empty((g * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out


def run_dist(gen, group=None):
    """Drive one rank's frame generator with torch.distributed collectives."""
    try:
        op = next(gen)
        while True:
            if isinstance(op, Exchange):
                op = gen.send(_a2a_dist(op, group))
            elif isinstance(op, AllGather):
                op = gen.send(_all_gather_dist(op, group))
            elif isinstance(op, ReduceScatter):
                op = gen.send(_reduce_scatter_dist(op, group))
            else:
                raise TypeError(f"unknown collective {op!r}")
    except StopIteration as e:
        return e.value


def run_loopback(gens: list):
    """Drive G frame generators (virtual ranks, one process) in lockstep."""
    G = len(gens)
    ops = [next(g) for g in gens]
    results = [None] * G
    while True:
        kinds = {type(o) for o in ops}
        if len(kinds) != 1:
            raise RuntimeError(f"ranks disagree on the collective: {kinds}")
        if isinstance(ops[0], AllGather):
            total = torch.cat([o.tensor for o in ops])
            outs = [total.clone() for _ in range(G)]
        elif isinstance(ops[0], Exchange):
            outs = []
            for r in range(G):
                parts = []
                for p in range(G):
                    if int(ops[r].recv_rows[p]) != int(ops[p].send_rows[r]):
                        raise RuntimeError("exchange row counts disagree")
                    off = int(sum(ops[p].send_rows[:r]))
                    parts.append(ops[p].tensor[off:off + int(ops[p].send_rows[r])])
                outs.append(torch.cat(parts) if parts else ops[r].tensor[:0])
        else:
            total = torch.stack([o.tensor for o in ops]).sum(0)
            rows = total.shape[0] // G
            outs = [total[r * rows:(r + 1) * rows].clone() for r in range(G)]
        nxt, done = [], 0
        for r, g in enumerate(gens):
            try:
                nxt.append(g.send(outs[r]))
            except StopIteration as e:
                results[r] = e.value
                nxt.append(None)
                done += 1
        if done == G:
            return results
        if done:
            raise RuntimeError("ranks finished at different collectives")
        ops = nxt
