"""The reference's vectorised key stages (src/keys.py:245-300) and stream helpers
(src/tracer.py:86-101) through the device implementation, bit-exact against fixtures
the reference produced (tests/golden/stages.npz, make_golden.py gen_stages)."""

import numpy as np
import pytest
import torch

from conftest import golden_cfg, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stages():
    return load_golden("stages.npz")


def _cfg(gpu, d, key):
    return gpu.FilterConfig(**golden_cfg(d, key))


def test_levels_array(gpu, stages):
    got = gpu.levels_array(stages["camera_distance"], _cfg(gpu, stages, "cfg"))
    assert np.array_equal(got.cpu().numpy(), stages["levels"])


def test_tangent_basis_array(gpu, stages):
    t1, t2 = gpu.tangent_basis_array(stages["normal"])
    assert np.array_equal(t1.cpu().numpy(), stages["t1"], equal_nan=True)
    assert np.array_equal(t2.cpu().numpy(), stages["t2"], equal_nan=True)


@pytest.mark.parametrize("which", ["jittered", "jittered_lv0"])
def test_jittered_positions(gpu, stages, which):
    cfg = _cfg(gpu, stages, "cfg")
    lv = stages["levels"] if which == "jittered" else np.zeros(len(stages["levels"]), np.int64)
    got = gpu.jittered_positions(stages["position"], stages["normal"], lv, stages["u1"],
                                 stages["u2"], cfg)
    assert np.array_equal(got.cpu().numpy(), stages[which], equal_nan=True)


def test_jitter_off_returns_positions(gpu, stages):
    cfg = _cfg(gpu, stages, "cfg")
    cfg.jitter = False
    got = gpu.jittered_positions(stages["position"], stages["normal"], stages["levels"],
                                 stages["u1"], stages["u2"], cfg)
    assert np.array_equal(got.cpu().numpy(), stages["position"])


@pytest.mark.parametrize("bins", [1, 2, 6, 8, 16, 64])
def test_normal_bins_array(gpu, stages, bins):
    got = gpu.normal_bins_array(stages["normal"], bins)
    assert np.array_equal(got.cpu().numpy(), stages[f"bins_{bins}"])


@pytest.mark.parametrize("key", ["cfg", "cfg_nfp"])
def test_aux_bits_array(gpu, stages, key):
    got = gpu.aux_bits_array(stages["normal"], stages["omega_r"], stages["layer_id"],
                             _cfg(gpu, stages, key))
    want = stages["aux" if key == "cfg" else "aux_nfp"]
    assert np.array_equal(got.cpu().numpy().astype(np.uint64), want)


def test_stream_descriptor_concat_select(gpu):
    from conftest import golden_stream
    d = load_golden("frame_box4.npz")
    host = golden_stream(d)
    vs = gpu.VertexStream.from_any(host)
    i = len(host.pixel) // 3
    desc = vs.descriptor(i)
    assert isinstance(desc, gpu.VertexDescriptor)
    assert np.array_equal(desc.position, host.position[i])
    assert desc.pixel == int(host.pixel[i]) and desc.sample == int(host.sample[i])
    assert desc.path_id == (int(host.sample[i]) << 32) | int(host.pixel[i])
    assert desc.camera_distance == float(host.camera_distance[i])
    mask = host.layer_id == 1
    sel = vs.select(mask)
    assert np.array_equal(sel.pixel.cpu().numpy(), host.pixel[mask])
    sel_t = vs.select(torch.as_tensor(mask, device="cuda"))
    assert torch.equal(sel_t.position, sel.position)
    both = gpu.VertexStream.concat([vs, sel])
    assert len(both) == len(vs) + len(sel)
    assert torch.equal(both.position[len(vs):], sel.position)
    assert len(gpu.VertexStream.concat([])) == 0


def test_backend_names(gpu):
    assert gpu.available_backends() == [gpu.BACKEND]
    from paper_1902_05942_b200._backend import get_kernels
    assert get_kernels(None) is get_kernels("native")
    with pytest.raises(ValueError):
        get_kernels("python")
    scene = gpu.closed_box(8, 8)
    with pytest.raises(ValueError):
        gpu.trace(scene, 1, 1, backend="python")
    a = gpu.trace(scene, 1, 1, threads=4)
    b = gpu.trace(scene, 1, 1, None, 1, 0, False, "native")
    assert torch.equal(a.image, b.image)


@pytest.mark.parametrize("delta", [0, 2])
def test_keys_across_lod_thresholds(gpu, stages, delta):
    """Jittered distances that do and do not cross a LOD threshold (about half of the
    rows change level): the kernel's threshold-distance shortcut (pf_config.lod_dist)
    must give the reference's keys bit for bit, including at d_k itself, 0, 1e300, inf."""
    cfg = _cfg(gpu, stages, "cfg")
    k = gpu.make_key_arrays(stages["near_position"], stages["near_normal"],
                            stages["near_normal"], stages["near_layer"],
                            stages["near_distance"], cfg, stages["near_u1"], stages["near_u2"],
                            delta).numpy()
    for f in ("qx", "qy", "qz", "level", "aux", "index", "fingerprint"):
        assert np.array_equal(k[f], stages[f"near{delta}_{f}"]), f
    assert np.array_equal(k["jittered"], stages[f"near{delta}_jittered"], equal_nan=True)

