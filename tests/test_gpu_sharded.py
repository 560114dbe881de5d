"""GPU parity of the key-sharded multi-GPU frame.

G virtual ranks run in one process on one device (`run_loopback`: every collective
is served in lockstep from the ranks' own buffers, no kernel waits on another
rank), so the sharded kernels, wire formats and host protocol are checked against
the single-GPU frame over the ranks' concatenated vertex streams.  Bar: identical
per-key table contents (the union of the owners' slices), bit-exact sources and
fixed-point means, images within float-atomic reordering."""

import numpy as np
import pytest
import torch

from test_gpu_parity import canon

pytestmark = pytest.mark.gpu


def _cat(parts):
    return {k: torch.cat([p[k] for p in parts]).contiguous() for k in parts[0]}


def _split_rows(stream, width, height, world):
    """Partition a stream by image row bands (band composite)."""
    rows = height // world
    out = []
    for r in range(world):
        lo, hi = r * rows * width, (r + 1) * rows * width
        m = (stream["pixel"] >= lo) & (stream["pixel"] < hi)
        out.append({k: v[m].contiguous() for k, v in stream.items()})
    return out


def _band_order(stream, width, height, world):
    """Rows of the full stream in the order of the concatenated band partitions."""
    rows = height // world
    px = stream["pixel"]
    return torch.cat([torch.nonzero((px >= r * rows * width) &
                                    (px < (r + 1) * rows * width)).reshape(-1)
                      for r in range(world)])


def _union_canon(states, table):
    rows = []
    for st in states:
        t = st.fine if table == "fine" else st.coarse
        rows += canon(t.state())
    return sorted(rows)


def _single(gpu, stream, base, cfg, spp, seed, frames=1):
    state = gpu.FrameState.from_config(cfg)
    outs = []
    for f in range(frames):
        vs = gpu.VertexStream(**stream)
        outs.append(gpu.filter_frame(vs, base, cfg, state, spp, seed + f))
    return state, outs


def _box(w, h, bounces, seed):
    from paper_1902_05942_b200.streams import camera_footprint, closed_box_stream
    s, base = closed_box_stream(w, h, bounces, seed)
    return s, base, camera_footprint(h)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("sum_mode", ["fixed", "float"])
def test_band_frame_matches_single(gpu, world, sum_mode):
    from paper_1902_05942_b200 import sharded
    w, h = 96, 64
    s, base, fs = _box(w, h, 4, 5)
    cap = 1 << (2 * w * h - 1).bit_length()
    cfg = gpu.FilterConfig(capacity=cap, footprint_scale=fs, sum_mode=sum_mode)
    single, [(img1, rep1, _)] = _single(gpu, s, base, cfg, 1, 11)
    parts = _split_rows(s, w, h, world)
    rows = h // world
    states = [sharded.ShardedState(cfg, r, world) for r in range(world)]
    gens = [sharded.filter_frame_sharded(gpu.VertexStream(**parts[r]),
                                         base[r * rows:(r + 1) * rows].contiguous(), cfg,
                                         states[r], 1, 11, pixel_base=r * rows * w)
            for r in range(world)]
    outs = sharded.run_loopback(gens)
    rtol = 1e-12 if sum_mode == "float" else 0.0
    for table in ("fine", "coarse"):
        a, b = _union_canon(states, table), canon(getattr(single, table).state())
        assert len(a) == len(b)
        for ra, rb in zip(a, b):
            assert ra[:4] == rb[:4]
            if rtol:
                np.testing.assert_allclose(ra[4] + ra[5], rb[4] + rb[5], rtol=rtol, atol=0)
            else:
                assert ra[4:] == rb[4:]
    # per-vertex results in the single run's order: row bands are pixel-ordered slices
    order = _band_order(s, w, h, world)
    src = torch.cat([o[1].source for o in outs])
    chosen = torch.cat([o[1].means for o in outs])
    assert torch.equal(src, rep1.source[order])
    if sum_mode == "fixed":
        assert torch.equal(chosen, rep1.means[order])
    else:
        torch.testing.assert_close(chosen, rep1.means[order], rtol=1e-12, atol=1e-300)
    img = torch.cat([o[0] for o in outs])
    torch.testing.assert_close(img, img1, rtol=1e-12, atol=1e-14)
    n_fine = sum(int(o[1].counters[gpu._lib.STAT_SOURCE_FINE]) +
                 int(o[1].counters[gpu._lib.STAT_SOURCE_NEIGHBORHOOD]) +
                 int(o[1].counters[gpu._lib.STAT_SOURCE_COARSE]) +
                 int(o[1].counters[gpu._lib.STAT_SOURCE_UNFILTERED]) for o in outs)
    assert n_fine == int(s["pixel"].shape[0])


@pytest.mark.parametrize("world", [2, 4])
def test_reduce_frame_multi_sample_matches_single(gpu, world):
    """Ranks trace different samples of the same pixels; the flat buffers are summed by
    a reduce-scatter and every rank returns its block of image rows."""
    from paper_1902_05942_b200 import sharded
    w, h, bounces = 64, 48, 3
    parts = []
    base = None
    for r in range(world):
        s, b, fs = _box(w, h, bounces, 100 + r)
        s["sample"] = s["sample"] + r * bounces
        parts.append(s)
        base = b if base is None else base
    cap = 1 << (2 * w * h - 1).bit_length()
    cfg = gpu.FilterConfig(capacity=cap, footprint_scale=fs, temporal_mode="filter")
    full = _cat(parts)
    single, frames1 = _single(gpu, full, base, cfg, world, 21, frames=3)
    states = [sharded.ShardedState(cfg, r, world) for r in range(world)]
    for f in range(3):
        gens = [sharded.filter_frame_sharded(gpu.VertexStream(**parts[r]), base, cfg, states[r],
                                             world, 21 + f, composite="reduce")
                for r in range(world)]
        outs = sharded.run_loopback(gens)
        img1, rep1, _ = frames1[f]
        assert torch.equal(torch.cat([o[1].source for o in outs]), rep1.source)
        torch.testing.assert_close(torch.cat([o[1].means for o in outs]), rep1.means,
                                   rtol=1e-13, atol=1e-300)
        torch.testing.assert_close(torch.cat([o[0] for o in outs]), img1, rtol=1e-12, atol=1e-14)
    for table in ("fine", "coarse"):
        a, b = _union_canon(states, table), canon(getattr(single, table).state())
        assert len(a) == len(b)
        for ra, rb in zip(a, b):
            assert ra[:4] == rb[:4]
            np.testing.assert_allclose(ra[4] + ra[5], rb[4] + rb[5], rtol=1e-12, atol=0)


def test_aggregation_overflow_regrows(gpu):
    """A tiny aggregation table overflows; the rank grows it, the ranks redo the count
    exchange in lockstep and still match the single-GPU frame."""
    from paper_1902_05942_b200 import sharded
    w, h = 64, 32
    s, base, fs = _box(w, h, 2, 9)
    cap = 1 << (2 * w * h - 1).bit_length()
    cfg = gpu.FilterConfig(capacity=cap, footprint_scale=fs, low_count_threshold=64)
    single, [(img1, rep1, _)] = _single(gpu, s, base, cfg, 1, 4)
    parts = _split_rows(s, w, h, 2)
    states = [sharded.ShardedState(cfg, r, 2, agg_capacity=64 if r == 0 else 1 << 16)
              for r in range(2)]
    gens = [sharded.filter_frame_sharded(gpu.VertexStream(**parts[r]),
                                         base[r * 16:(r + 1) * 16].contiguous(), cfg, states[r],
                                         1, 4, pixel_base=r * 16 * w) for r in range(2)]
    outs = sharded.run_loopback(gens)
    assert states[0].regrows >= 1  # the records outgrew 64 slots
    order = _band_order(s, w, h, 2)
    assert torch.equal(torch.cat([o[1].source for o in outs]), rep1.source[order])
    assert torch.equal(torch.cat([o[1].means for o in outs]), rep1.means[order])


def test_bad_input_rejected_on_every_rank(gpu):
    from paper_1902_05942_b200 import sharded
    w, h = 32, 16
    s, base, fs = _box(w, h, 2, 3)
    cfg = gpu.FilterConfig(capacity=2048, footprint_scale=fs)
    parts = _split_rows(s, w, h, 2)
    parts[1]["contribution"][5, 1] = float("nan")
    states = [sharded.ShardedState(cfg, r, 2) for r in range(2)]
    gens = [sharded.filter_frame_sharded(gpu.VertexStream(**parts[r]),
                                         base[r * 8:(r + 1) * 8].contiguous(), cfg, states[r], 1,
                                         1, pixel_base=r * 8 * w) for r in range(2)]
    with pytest.raises(ValueError):
        sharded.run_loopback(gens)
    for st in states:
        assert st.fine.total_counts() == 0 and st.coarse.total_counts() == 0
        assert int(st.n_distinct.item()) == 0


def test_shard_abi_rejects_bad_geometry(gpu):
    from paper_1902_05942_b200 import sharded
    cfg = gpu.FilterConfig(capacity=1024)
    with pytest.raises(ValueError):
        sharded.ShardedState(cfg, 0, 3)
    with pytest.raises(ValueError):
        sharded.ShardedState(cfg, 2, 2)
    st = sharded.ShardedState(cfg, 1, 2)
    st.world = 2
    sh = st.c_shard()
    sh.log2_capacity = 30
    import ctypes
    with pytest.raises(ValueError):
        gpu._lib.call("pf_shard_reset", ctypes.byref(sh), gpu._lib.stream_handle())


def _dist_worker(rank, world, port, out_dir):
    import os
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1902_05942_b200 as pf
        from paper_1902_05942_b200 import sharded
        w, h = 64, 32
        s, base, fs = _box(w, h, 3, 40 + rank)
        s["sample"] = s["sample"] + 3 * rank
        base = _box(w, h, 1, 1)[1]
        cfg = pf.FilterConfig(capacity=4096, footprint_scale=fs)
        st = sharded.ShardedState(cfg, rank, world)
        img, rep, _ = sharded.run_dist(sharded.filter_frame_sharded(
            pf.VertexStream(**s), base, cfg, st, world, 7, composite="reduce"))
        torch.save({"image": img.cpu(), "source": rep.source.cpu(), "means": rep.means.cpu()},
                   os.path.join(out_dir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_run_dist_gloo_two_processes(gpu, tmp_path):
    """The torch.distributed driver with real frame tensors: two processes on one
    device exchange through gloo (host memory; no kernel waits on another process)
    and reproduce the single-GPU frame over both streams."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_dist_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    res = [torch.load(tmp_path / f"rank{r}.pt") for r in range(2)]
    w, h = 64, 32
    parts = []
    for r in range(2):
        s, _, fs = _box(w, h, 3, 40 + r)
        s["sample"] = s["sample"] + 3 * r
        parts.append(s)
    base = _box(w, h, 1, 1)[1]
    cfg = gpu.FilterConfig(capacity=4096, footprint_scale=fs)
    _, [(img1, rep1, _)] = _single(gpu, _cat(parts), base, cfg, 2, 7)
    assert torch.equal(torch.cat([r["source"] for r in res]), rep1.source.cpu())
    assert torch.equal(torch.cat([r["means"] for r in res]), rep1.means.cpu())
    torch.testing.assert_close(torch.cat([r["image"] for r in res]), img1.cpu(), rtol=1e-12,
                               atol=1e-14)


def test_rank_without_vertices(gpu):
    """A rank whose band traced nothing still takes part in every collective."""
    from paper_1902_05942_b200 import sharded
    w, h = 32, 16
    s, base, fs = _box(w, h, 2, 6)
    cfg = gpu.FilterConfig(capacity=2048, footprint_scale=fs)
    parts = _split_rows(s, w, h, 2)
    parts[1] = {k: v[:0] for k, v in parts[1].items()}
    single, [(img1, rep1, _)] = _single(gpu, parts[0], base, cfg, 1, 2)
    states = [sharded.ShardedState(cfg, r, 2) for r in range(2)]
    gens = [sharded.filter_frame_sharded(gpu.VertexStream(**parts[r]),
                                         base[r * 8:(r + 1) * 8].contiguous(), cfg, states[r], 1,
                                         2, pixel_base=r * 8 * w) for r in range(2)]
    outs = sharded.run_loopback(gens)
    assert torch.equal(outs[0][1].source, rep1.source)
    assert torch.equal(outs[1][0], base[8:])
    torch.testing.assert_close(outs[0][0], img1[:8], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("name", ["aux", "delta3", "nfp", "nojit", "single", "thr1", "thr64"])
def test_variants_sharded_match_reference(gpu, name):
    """The key / ladder options of frame_variants.npz through the 2-rank sharded frame
    (pixel row bands of 14 and 13 rows, band composite): the reference's sources,
    means, image and per-key tables."""
    from conftest import golden_cfg, golden_stream, golden_table, load_golden
    from paper_1902_05942_b200 import sharded
    d = load_golden("frame_variants.npz")
    vs = gpu.VertexStream.from_any(golden_stream(d))
    cfg = gpu.FilterConfig(**golden_cfg(d, f"{name}_cfg"))
    base = torch.as_tensor(d["base"], device="cuda")
    H, W = int(base.shape[0]), int(base.shape[1])
    world, split = 2, 14
    bands = [(0, split), (split, H)]
    rows = [torch.nonzero((vs.pixel >= a * W) & (vs.pixel < b * W)).reshape(-1) for a, b in bands]
    states = [sharded.ShardedState(cfg, r, world) for r in range(world)]
    outs = sharded.run_loopback([sharded.filter_frame_sharded(
        vs.select(rows[r]), base[a:b].contiguous(), cfg, states[r], int(d["spp"]),
        int(d["seed"]), pixel_base=a * W) for r, (a, b) in enumerate(bands)])
    order = torch.cat(rows).cpu().numpy()
    assert np.array_equal(torch.cat([o[1].source for o in outs]).cpu().numpy(),
                          d[f"{name}_source"][order])
    means = torch.cat([o[1].means for o in outs]).cpu().numpy()
    if cfg.sum_mode == "float":
        np.testing.assert_allclose(means, d[f"{name}_chosen"][order], rtol=1e-12, atol=0)
    else:
        assert np.array_equal(means, d[f"{name}_chosen"][order])
    img = torch.cat([o[0] for o in outs]).cpu().numpy()
    np.testing.assert_allclose(img, d[f"{name}_image"], rtol=1e-12, atol=1e-300)
    tables = ("fine", "coarse") if cfg.multi_level else ("fine",)
    for table in tables:
        a = _union_canon(states, table)
        b = canon(golden_table(d, f"{name}_{table}_"))
        assert len(a) == len(b)
        for ra, rb in zip(a, b):
            assert ra[:4] == rb[:4]
            if cfg.sum_mode == "float":
                np.testing.assert_allclose(ra[4] + ra[5], rb[4] + rb[5], rtol=1e-12, atol=0)
            else:
                assert ra[4:] == rb[4:]
