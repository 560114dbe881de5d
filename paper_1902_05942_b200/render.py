"""Whole frames on the device: trace -> temporal update -> accumulate -> (hybrid replay)
-> resolve (src/pipeline.py:286-380: render_frame, run_sequence,
_apply_temporal_differences).

The tracer (csrc/pf_trace.cu) writes the vertex stream straight into HBM, so a frame
never touches the host.  integrate / filter frames run the fused pf_filter_frame call;
hybrid frames run the phases separately because the replay of a round-robin slice of
last frame's paths (reevaluate) must land its per-voxel deltas between accumulate and
resolve, as in the reference.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from . import rng
from .keys import FilterConfig
from .pipeline import FrameState, FrameStats, ResolveReport, accumulate_phase, filter_frame, \
    resolve_phase
from .scene import Scene
from .temporal import reevaluation_deltas, select_replay_ids
from .tracer import TraceOptions, TraceResult, reevaluate, trace


@dataclass
class FrameResult:
    """src/pipeline.py:108-116 (device tensors)."""

    filtered: torch.Tensor
    unfiltered: torch.Tensor
    stats: FrameStats
    report: ResolveReport
    trace_result: TraceResult
    fine_keys: object
    coarse_keys: object


def _intersect_sorted(a: torch.Tensor, b: torch.Tensor):
    """np.intersect1d(a, b, return_indices=True) for arrays of unique values."""
    sa, ia = torch.sort(a)
    sb, ib = torch.sort(b)
    keep = torch.isin(sa, sb)
    common = sa[keep]
    return common, ia[keep], ib[torch.searchsorted(sb, common)]


def apply_temporal_differences(scene_f: Scene, cfg: FilterConfig, state: FrameState, frame: int,
                               options: TraceOptions | None = None):
    """Replay a slice of last frame's paths and store per-cell deltas (src/pipeline.py:286-318)."""
    prev = getattr(state, "prev_vertices", None)
    if prev is None or len(prev) == 0:
        return
    ids = prev.path_id
    chosen = select_replay_ids(ids, frame, cfg.reevaluate_fraction)
    if chosen.numel() == 0:
        return
    rows = torch.nonzero(torch.isin(ids, chosen)).reshape(-1)
    replay = reevaluate(scene_f, state.prev_seed, state.prev_spp, ids[rows], options)
    if len(replay) == 0:  # moving geometry can lose every replayed vertex
        return
    common, orig_pos, re_pos = _intersect_sorted(ids[rows], replay.path_id)
    if common.numel() == 0:
        return
    rows = rows[orig_pos]
    replay = replay.select(re_pos)
    orig = prev.select(rows)
    for table, keys in ((state.fine, state.prev_fine_keys),
                        (state.coarse, state.prev_coarse_keys)):
        if table is None or keys is None:
            continue
        idx, fp, deltas = reevaluation_deltas(orig, replay, keys.qx[rows], keys.qy[rows],
                                              keys.qz[rows], keys.level[rows], keys.aux[rows],
                                              cfg)
        slots = table.lookup_slots(idx, fp)
        ok = slots >= 0
        table.set_deltas(slots[ok], deltas[ok])


def render_frame(scene: Scene, cfg: FilterConfig, state: FrameState, spp: int, seed: int,
                 threads: int = 1, options: TraceOptions | None = None,
                 backend: str | None = None) -> FrameResult:
    """Trace, begin the generation, accumulate, resolve, advance (src/pipeline.py:321-363).
    `threads` only names the reference's tracer parallelism (see tracer.trace)."""
    t0 = time.perf_counter()
    frame = state.frame
    scene_f = scene.at_frame(frame)
    cfg_f = cfg.for_camera(scene_f.camera.fov, scene_f.camera.height)
    frame_seed = rng.frame_seed(seed, frame) if scene.frames > 1 else seed
    t1 = time.perf_counter()
    tr = trace(scene_f, spp, frame_seed, options, backend=backend)
    t2 = time.perf_counter()
    if cfg.temporal_mode == "hybrid":
        state.fine.begin_frame(frame, cfg_f)
        if state.coarse is not None:
            state.coarse.begin_frame(frame, cfg_f)
        fine_keys, coarse_keys, stats = accumulate_phase(tr.vertices, cfg_f, state, frame,
                                                         frame_seed)
        apply_temporal_differences(scene_f, cfg_f, state, frame, options)
        t3 = time.perf_counter()
        filtered, report = resolve_phase(tr.vertices, cfg_f, state, frame, frame_seed, spp,
                                         tr.base_image, fine_keys)
        state.prev_fine_keys, state.prev_coarse_keys = fine_keys, coarse_keys
        state.prev_seed, state.prev_spp, state.frame = frame_seed, spp, frame + 1
    else:
        filtered, report, stats = filter_frame(tr.vertices, tr.base_image, cfg_f, state, spp,
                                               frame_seed)
        fine_keys, coarse_keys = state.prev_fine_keys, state.prev_coarse_keys
        t3 = time.perf_counter()
    t4 = time.perf_counter()
    stats.evictions = len(state.fine.eviction_events)
    stats.horizon_clears = state.fine.horizon_clears
    stats.occupancy_fine = state.fine.occupancy()
    stats.occupancy_coarse = state.coarse.occupancy() if state.coarse is not None else 0.0
    stats.source_counts = report.counts
    stats.time_trace, stats.time_accumulate = t2 - t1, t3 - t2
    stats.time_resolve, stats.time_total = t4 - t3, t4 - t0
    state.prev_vertices = tr.vertices
    return FrameResult(filtered, tr.image, stats, report, tr, fine_keys, coarse_keys)


def run_sequence(scene: Scene, cfg: FilterConfig, spp: int, seed: int, frames: int | None = None,
                 threads: int = 1, options: TraceOptions | None = None,
                 backend: str | None = None, on_frame=None, ordered: bool = False) -> list:
    """`frames` frames with persistent temporal state (src/pipeline.py:366-380).
    ordered=True uses sequential-order tables (the reference's threads=1 slot layout)."""
    cfg = cfg.for_camera(scene.camera.fov, scene.camera.height)
    state = FrameState.from_config(cfg, ordered=ordered)
    out = []
    for _ in range(frames if frames is not None else scene.frames):
        res = render_frame(scene, cfg, state, spp, seed, threads, options, backend)
        out.append(res)
        if on_frame is not None:
            on_frame(res)
    return out
