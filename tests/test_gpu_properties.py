"""Property-based and statistical tests in the style of the reference's own suite
(pkg/tests/test_keys.py:63-68, 100-109, 153-166, 242-267;
test_rng.py:25-32; test_table.py:96-120), run against the device kernels."""

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu


def _stream(n, seed, spread=50.0):
    r = np.random.default_rng(seed)
    nrm = r.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    om = r.normal(size=(n, 3))
    om /= np.linalg.norm(om, axis=1, keepdims=True)
    return dict(position=r.uniform(-spread, spread, (n, 3)), normal=nrm, omega_r=om,
                contribution=r.uniform(0.0, 4.0, (n, 3)), throughput=np.ones((n, 3)),
                pixel=r.integers(0, 1 << 20, n), sample=r.integers(0, 4, n),
                layer_id=r.integers(0, 3, n), camera_distance=r.uniform(0.5, 200.0, n))


@settings(max_examples=25, deadline=None)
@given(st.lists(st.floats(min_value=1e-3, max_value=1e6, allow_nan=False), min_size=2,
                max_size=64))
def test_lod_is_monotone_in_distance(gpu, dists):
    """Farther vertices never get a finer level (test_keys.py:63-68)."""
    d = np.sort(np.asarray(dists, np.float64))
    n = len(d)
    z3 = np.zeros((n, 3))
    nrm = np.tile([0.0, 0.0, 1.0], (n, 1))
    cfg = gpu.FilterConfig(capacity=1024, jitter=False, footprint_scale=0.0013)
    k = gpu.make_key_arrays(z3, nrm, nrm, np.zeros(n, np.int64), d, cfg).numpy()
    assert np.all(np.diff(k["level"]) >= 0)
    assert k["level"].min() >= 0 and k["level"].max() <= 31


@settings(max_examples=20, deadline=None)
@given(st.integers(-2**40, 2**40), st.integers(-2**40, 2**40), st.integers(-2**40, 2**40),
       st.integers(0, 31), st.integers(0, 2**26))
def test_equal_keys_hash_equally(gpu, qx, qy, qz, lv, aux):
    """The hash is a function of the key fields (test_keys.py:153-166): equal keys give
    equal (index, fingerprint), a changed field almost surely changes them."""
    a = gpu.hashes(gpu.CellKey(qx, qy, qz, lv, aux))
    b = gpu.hashes(gpu.CellKey(qx, qy, qz, lv, aux))
    c = gpu.hashes(gpu.CellKey(qx + 1, qy, qz, lv, aux))
    assert (a.index, a.fingerprint) == (b.index, b.fingerprint)
    assert (a.index, a.fingerprint) != (c.index, c.fingerprint)
    assert a.fingerprint != 0  # the sentinel is remapped (src/keys.py:214-215)


def test_home_slots_are_uniform(gpu):
    """Poisson slot occupancy: a chi-square test of home slots over 2^12 buckets for
    2^20 distinct keys (test_keys.py:242-267)."""
    from scipy.stats import chisquare
    n = 1 << 20
    q = torch.arange(n, dtype=torch.int64, device="cuda")
    z = torch.zeros_like(q)
    idx, _ = gpu.hash_arrays(q % 1024, q // 1024, z, z + 3, z)
    buckets = 1 << 12
    counts = torch.bincount((idx & (buckets - 1)), minlength=buckets).cpu().numpy()
    assert chisquare(counts).pvalue > 1e-4


def test_jitter_is_centred(gpu):
    """Disc jitter has mean ~0 within 3 sigma in both tangent directions and stays inside
    half a voxel (test_keys.py:100-109), from the device RNG."""
    n = 1 << 18
    vs = _stream(n, 4)
    vs["position"] = np.tile([1.5, 2.5, 3.5], (n, 1))
    vs["normal"] = np.tile([0.0, 0.0, 1.0], (n, 1))
    vs["camera_distance"] = np.full(n, 3.0)
    vs["pixel"] = np.arange(n)
    vs["sample"] = np.zeros(n, np.int64)
    cfg = gpu.FilterConfig(capacity=1024, footprint_scale=0.001)
    k = gpu.vertex_keys(gpu.VertexStream.from_any(type("S", (), vs)()), cfg, 17).numpy()
    off = k["jittered"] - vs["position"]
    half = cfg.voxel_size(int(k["level"][0])) / 2
    assert np.all(np.hypot(off[:, 0], off[:, 1]) <= half * (1 + 1e-12))
    assert np.all(off[:, 2] == 0.0)
    for c in (0, 1):
        sigma = off[:, c].std() / np.sqrt(n)
        assert abs(off[:, c].mean()) < 3 * sigma


def test_jitter_streams_are_decorrelated(gpu):
    """Accumulate (stream 2) and lookup (stream 3) jitter are uncorrelated
    (test_rng.py:25-32)."""
    n = 1 << 18
    vs = _stream(n, 5)
    vs["normal"] = np.tile([0.0, 0.0, 1.0], (n, 1))
    vs["pixel"] = np.arange(n)
    cfg = gpu.FilterConfig(capacity=1024, footprint_scale=0.001)
    v = gpu.VertexStream.from_any(type("S", (), vs)())
    a = gpu.vertex_keys(v, cfg, 9, 2).numpy()["jittered"] - vs["position"]
    b = gpu.vertex_keys(v, cfg, 9, 3).numpy()["jittered"] - vs["position"]
    r = np.corrcoef(a[:, 0], b[:, 0])[0, 1]
    assert abs(r) < 4 / np.sqrt(n)


@pytest.mark.parametrize("sum_mode", ["fixed", "float"])
def test_conservation_across_seeds(gpu, sum_mode):
    """Every vertex lands in exactly one cell: counts and (fixed-point exact) sums are
    conserved under the massively parallel insert, 10 seeds (test_table.py:96-120)."""
    for seed in range(10):
        r = np.random.default_rng(seed)
        n = 50000
        idx = r.integers(0, 2**63, 700).astype(np.uint64)[r.integers(0, 700, n)]
        fp = ((idx >> np.uint64(7)) & np.uint64(0xFFFFFFFF)).astype(np.uint32) | np.uint32(1)
        vals = r.uniform(0.0, 3.0, (n, 3))
        t = gpu.VoxelTable(4096, sum_mode=sum_mode)
        st_, _, _ = t.accumulate_batch(idx, fp, vals, 0)
        assert int((st_ == 2).sum()) == 0
        assert t.total_counts() == n
        if sum_mode == "fixed":
            want = np.floor(vals * 65536.0 + 0.5).astype(np.int64).sum(0)
            assert np.array_equal(t.sums.sum(0).cpu().numpy(), want)
        else:
            np.testing.assert_allclose(t.sums.sum(0).cpu().numpy(), vals.sum(0), rtol=1e-12)


def test_conservation_large_fixed_values(gpu):
    """Quanta at and above 2^27 (contributions >= 2048) take the pointer-jumping group sum
    instead of the 32-bit warp reduction; sums stay exact, mixed per warp."""
    r = np.random.default_rng(77)
    n = 40000
    idx = r.integers(0, 2**63, 300).astype(np.uint64)[r.integers(0, 300, n)]
    fp = ((idx >> np.uint64(7)) & np.uint64(0xFFFFFFFF)).astype(np.uint32) | np.uint32(1)
    vals = r.uniform(0.0, 3.0, (n, 3))
    big = r.uniform(size=n) < 0.05
    vals[big] = r.uniform(2047.0, 1e6, (int(big.sum()), 3))
    vals[:32] = (2.0 ** 27 - 1) / 65536.0  # quanta 2^27 - 1 (fast path) and 2^27 (not)
    vals[32:64] = 2048.0
    t = gpu.VoxelTable(1024, sum_mode="fixed")
    st_, _, _ = t.accumulate_batch(idx, fp, vals, 0)
    assert int((st_ == 2).sum()) == 0
    assert t.total_counts() == n
    want = np.floor(vals * 65536.0 + 0.5).astype(np.int64).sum(0)
    assert np.array_equal(t.sums.sum(0).cpu().numpy(), want)
