"""GPU parity of the on-device path tracer (csrc/pf_trace.cu) against the reference
tracer's own output (tests/golden/tracer.npz, made by running src/tracer.py).

Bar: the same set of recorded paths (vertex selection, Russian roulette and
visibility decisions) and bit-identical vertex records -- the tracer computes in FP64
with numpy's operation order and glibc's sin/cos (csrc/pf_device.cuh: glibc_sincos).
Only the glossy lobe's pow is CUDA's (numpy's pow is its own SIMD routine), so the
glossy scene is compared with rtol 1e-9.  Images (sums over samples) within 1e-15.
The filter keys built from the traced stream must equal those of the reference's."""

import numpy as np
import pytest
import torch

from conftest import STREAM_FIELDS, golden_stream, load_golden

pytestmark = pytest.mark.gpu

CASES = {
    # name: (scene builder, spp, seed, options kwargs, rtol)
    "box_k1": (lambda S: S.closed_box(48, 27), 1, 1, dict(select_k=1, rr_start=9), 0.0),
    "box_k2": (lambda S: S.closed_box(48, 27), 1, 1, dict(select_k=2, rr_start=9), 0.0),
    "box_k3": (lambda S: S.closed_box(48, 27), 1, 1, dict(select_k=3, rr_start=9), 0.0),
    "box_k4": (lambda S: S.closed_box(48, 27), 1, 1, dict(select_k=4, rr_start=9), 0.0),
    "cornell": (lambda S: S.load_scene("cornell", 32, 32), 2, 5, {}, 0.0),
    "glossy": (lambda S: S.load_scene("cornell-glossy", 24, 24), 1, 3, dict(select_k=2), 1e-9),
    "sweep": (lambda S: S.load_scene("shadow-sweep", 24, 24).at_frame(3), 1, 7, {}, 0.0),
    "occluded": (lambda S: S.load_scene("occluded", 8, 8), 1, 2, {}, 0.0),
    "corridor": (lambda S: S.load_scene("corridor", 20, 16).at_frame(5), 1, 9,
                 dict(nee=False, pixel_jitter=False, max_depth=5), 0.0),
}


def _np(t):
    return t.cpu().numpy()


def _paths(pixel, sample):
    return (np.asarray(sample, np.int64) << 32) | np.asarray(pixel, np.int64)


def _compare_streams(got, want, rtol):
    gid, wid = _paths(_np(got.pixel), _np(got.sample)), _paths(want.pixel, want.sample)
    # the same paths recorded a vertex, in the same order
    assert np.array_equal(gid, wid), (len(gid), len(wid))
    for f in ("position", "normal", "omega_r", "throughput", "camera_distance", "contribution"):
        if rtol == 0.0:
            assert np.array_equal(_np(getattr(got, f)), getattr(want, f)), f
        else:  # glossy: pow differs by ulps; 1e-12 absolute floor for values near 0
            np.testing.assert_allclose(_np(getattr(got, f)), getattr(want, f), rtol=rtol,
                                       atol=1e-12, err_msg=f)
    assert np.array_equal(_np(got.layer_id), want.layer_id)


@pytest.mark.parametrize("name", list(CASES))
def test_trace_matches_reference(gpu, name):
    from paper_1902_05942_b200 import scene as S
    from paper_1902_05942_b200.tracer import TraceOptions, trace
    d = load_golden("tracer.npz")
    build, spp, seed, kw, rtol = CASES[name]
    res = trace(build(S), spp, seed, TraceOptions(**kw), want_variance=(name == "cornell"))
    _compare_streams(res.vertices, golden_stream(d, f"{name}_v_"), rtol)
    # per-pixel sums over samples are plain tensor adds in sample order, as numpy's
    np.testing.assert_allclose(_np(res.image), d[f"{name}_image"], rtol=rtol or 1e-15,
                               atol=1e-300)
    np.testing.assert_allclose(_np(res.base_image), d[f"{name}_base"], rtol=rtol or 1e-15,
                               atol=1e-300)
    if name == "cornell":
        np.testing.assert_allclose(_np(res.variance), d["cornell_variance"], rtol=1e-9,
                                   atol=1e-14)
    if name == "occluded":
        assert float(res.image.abs().max()) == 0.0


def test_reevaluate_replays_paths(gpu):
    from paper_1902_05942_b200 import scene as S
    from paper_1902_05942_b200.tracer import reevaluate, trace
    d = load_golden("tracer.npz")
    cb = S.load_scene("cornell", 32, 32)
    got = reevaluate(cb, 5, 2, d["reeval_ids"])
    _compare_streams(got, golden_stream(d, "reeval_v_"), 0.0)
    # a static scene replays the original trace's rows bit for bit
    full = trace(cb, 2, 5).vertices
    ids_full = _paths(_np(full.pixel), _np(full.sample))
    ids_re = _paths(_np(got.pixel), _np(got.sample))
    pos = {int(p): i for i, p in enumerate(ids_full)}
    rows = np.array([pos[int(p)] for p in ids_re])
    for f in STREAM_FIELDS:
        assert np.array_equal(_np(getattr(full, f))[rows], _np(getattr(got, f))), f
    with pytest.raises(ValueError):
        reevaluate(cb, 5, 2, np.array([1 << 40], np.uint64))


def test_traced_stream_keys_equal_reference_keys(gpu):
    """The whole point of tracing on the device: the filter's keys from the GPU-traced
    benchmark stream equal those of the reference's stream (same cells)."""
    from paper_1902_05942_b200 import scene as S
    from paper_1902_05942_b200.streams import camera_footprint
    from paper_1902_05942_b200.tracer import multi_bounce_stream
    d = load_golden("tracer.npz")
    vs, base = multi_bounce_stream(S.closed_box(48, 27), 4, 1)
    want = [golden_stream(d, f"box_k{k}_v_") for k in range(1, 5)]
    cfg = gpu.FilterConfig(capacity=4096, footprint_scale=camera_footprint(27))
    got_k = gpu.vertex_keys(vs, cfg, 11)
    ref_vs = gpu.VertexStream.from_any(type("S", (), {
        f: np.concatenate([getattr(w, f) + (k if f == "sample" else 0)
                           for k, w in enumerate(want)]) for f in STREAM_FIELDS})())
    want_k = gpu.vertex_keys(ref_vs, cfg, 11)
    for f in ("index", "fingerprint", "level", "qx", "qy", "qz"):
        assert torch.equal(getattr(got_k, f), getattr(want_k, f)), f


@pytest.mark.parametrize("world", [2, 4])
def test_band_stream_is_the_frame_stream_restricted_to_its_rows(gpu, world):
    """bench --workload uhd4-band: rank r's band_stream equals the whole frame's
    multi_bounce_stream restricted to the pixels of rows [r H/G, (r+1) H/G), field by
    field and in order; the band base image is those rows of the frame's base."""
    from paper_1902_05942_b200.scene import closed_box
    from paper_1902_05942_b200.tracer import band_stream, multi_bounce_stream
    w, h = 48, 28
    sc = closed_box(w, h)
    full, base = multi_bounce_stream(sc, 4, 1)
    rows = h // world
    for r in range(world):
        vs, b = band_stream(sc, 4, 1, r * rows, (r + 1) * rows)
        m = (full.pixel >= r * rows * w) & (full.pixel < (r + 1) * rows * w)
        for f in ("position", "normal", "omega_r", "contribution", "throughput", "pixel",
                  "sample", "layer_id", "camera_distance"):
            assert torch.equal(getattr(vs, f), getattr(full, f)[m]), f
        assert torch.equal(b, base[r * rows:(r + 1) * rows])
