"""begin_frame over the occupied-slot lists the previous fused frame left behind
(pf_frame_buffers.occ_*) must fold exactly what the tag sweep folds.

Two FrameStates run the same frames in lockstep: one uses the lists (the default), the
other is forced to sweep every frame.  Between frames the test also mutates the tables
through the API (accumulate_batch, set_deltas) and through an in-place tensor write, which
must invalidate the lists; sources, means, image and both tables (per key) stay
bit-identical throughout.
"""

import numpy as np
import pytest
import torch

from oracle.golden import golden_cfg, golden_stream, load_golden

pytestmark = pytest.mark.gpu


def _tables_equal(a, b):
    """Per key (order-free rows: the parallel insert's slot choice among racing claims is
    not deterministic, so slot positions may differ between two runs)."""
    from oracle.digest import table_digest
    for ta, tb in ((a.fine, b.fine), (a.coarse, b.coarse)):
        assert table_digest(ta.state()) == table_digest(tb.state())


@pytest.mark.parametrize("mode", ["integrate", "filter", "hybrid"])
def test_occupied_lists_match_sweep(gpu, mode):
    d = load_golden("frame_cornell128.npz")
    vs = golden_stream(d)
    cfgd = golden_cfg(d, "fixed_cfg")
    cfgd["temporal_mode"] = mode
    # no eviction pressure and no horizon clears within the 12 frames: with holes in the
    # probe chains, which of two racing claims takes a slot (run-dependent in the parallel
    # insert) decides later lookups, and two runs could differ whatever begin_frame does
    cfgd["capacity"] = 1 << 16
    cfgd["evict_horizon"] = 64
    cfg = gpu.FilterConfig(**cfgd)
    lists, sweep = gpu.FrameState.from_config(cfg), gpu.FrameState.from_config(cfg)
    n = len(vs.pixel)
    used = 0
    for f in range(12):
        # a shifted window of the stream each frame: cells leave it and age
        lo = (f * 1543) % (n // 2)
        sub = gpu.VertexStream.from_any(type("S", (), {
            k: getattr(vs, k)[lo:lo + n // 2] for k in (
                "position", "normal", "omega_r", "contribution", "throughput", "pixel",
                "sample", "layer_id", "camera_distance")})())
        sweep.scratch.pop("_occ_prev", None)   # force the tag sweep
        outs = []
        for st in (lists, sweep):
            if st is lists:
                from paper_1902_05942_b200.pipeline import _occ_key
                prev = st.scratch.get("_occ_prev")
                used += int(prev is not None and prev[0] == _occ_key(st))
            img, rep, _ = gpu.filter_frame(sub, d["base"], cfg, st, 1, 11 + f)
            outs.append((img.cpu().numpy(), rep.source.cpu().numpy(), rep.means.cpu().numpy()))
        for x, y in zip(outs[0], outs[1]):
            assert np.array_equal(x, y), f
        _tables_equal(lists, sweep)
        if f == 4:  # an API insert between frames on both (keys of cells that exist: no
            # new claims, whose racing slot choice would make the two runs' layouts differ)
            from paper_1902_05942_b200 import rng as prng
            from paper_1902_05942_b200.pipeline import vertex_keys
            k = vertex_keys(sub, cfg, 11 + f, prng.STREAM_JITTER_ACCUM, 0)
            idx, fp = k.index[:64], k.fingerprint[:64]
            vals = torch.rand((64, 3), dtype=torch.float64, device=idx.device,
                              generator=torch.Generator(device=idx.device).manual_seed(3))
            for st in (lists, sweep):
                st.fine.accumulate_batch(idx, fp, vals, f)
        if f == 7:  # an in-place tensor write on both (value unchanged, version bumped)
            for st in (lists, sweep):
                st.fine.deltas[0] = st.fine.deltas[0].clone()
    assert 8 <= used <= 9  # frames 1-11 fold from the lists except after the two mutations
    torch.cuda.synchronize()
