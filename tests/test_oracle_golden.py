"""Pin the CPU oracle to the reference: every golden fixture in tests/golden/ was
produced by the reference package itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import TABLE_FIELDS, golden_cfg, golden_stream, golden_table, load_golden

# pkg/tests/test_keys.py:195-205 -- the reference's frozen hash vectors
REFERENCE_GOLDEN_VECTORS = [
    ((0, 0, 0, 0, 0), 0x2B875FE90B264F7C, 0x88E2E49F),
    ((1, 0, 0, 0, 0), 0x8B9EAAC55FD6045E, 0x3C966E6F),
    ((-1, 2, -3, 0, 0), 0x6C23EDB01E685DFC, 0xCF566B5E),
    ((6, -3, 1, 0, 0), 0x85F8CCE9FA9EAD67, 0xFECBB755),
    ((123456, -654321, 42, 7, 0), 0x47B6C4C058225B54, 0x69258E3A),
    ((0, 0, 0, 31, 0), 0x7379FD7CE8144994, 0xCD3BFD50),
    ((5, 5, 5, 3, 16909060), 0x03E6656A1B359254, 0xC4EA312A),
    ((-1099511627776, 1099511627776, -7, 12, 63), 0x87CBB877676F99D4, 0x3B89422E),
]


def _cfg(oracle, d, key):
    c = golden_cfg(d, key)
    return oracle.Config(**{k: v for k, v in c.items() if k in oracle.Config.__dataclass_fields__})


def test_reference_hash_vectors(oracle):
    for (qx, qy, qz, lv, aux), index, fp in REFERENCE_GOLDEN_VECTORS:
        i, f = oracle.cell_hashes([qx], [qy], [qz], [lv], np.array([aux], np.uint64))
        assert int(i[0]) == index and int(f[0]) == fp


def test_sentinel_remap(oracle):
    # a fingerprint that hashes to the empty sentinel must come back as 1 (src/keys.py:338)
    _, f = oracle.cell_hashes([0], [0], [0], [0], np.zeros(1, np.uint64),
                              fp_bins=np.zeros(1, np.uint32))
    assert int(f[0]) != 0


def test_rng_draws(oracle):
    d = load_golden("rng_hash.npz")
    ids = d["draw_ids"]
    for si, seed in enumerate(d["draw_seeds"]):
        for stream in (1, 2, 3):
            for dim in (0, 1):
                got = oracle.draw_u64(int(seed), stream, ids, 0, dim)
                assert np.array_equal(got, d[f"draw_u64_{si}_{stream}_{dim}"])
                got = oracle.draw_unit(int(seed), stream, ids, 0, dim)
                assert np.array_equal(got, d[f"draw_unit_{si}_{stream}_{dim}"])


def test_hash_arrays(oracle):
    d = load_golden("rng_hash.npz")
    q = d["hq"]
    i, f = oracle.cell_hashes(q[:, 0], q[:, 1], q[:, 2], d["hlevel"], d["haux"])
    assert np.array_equal(i, d["hindex"]) and np.array_equal(f, d["hfp"])
    i, f = oracle.cell_hashes(q[:, 0], q[:, 1], q[:, 2], d["hlevel"], d["haux"], d["hbins"])
    assert np.array_equal(i, d["hindex_b"]) and np.array_equal(f, d["hfp_b"])


@pytest.mark.parametrize("variant", ["default", "aux", "nfp", "nojit"])
def test_keys_random(oracle, variant):
    d = load_golden("keys_random.npz")
    vs = golden_stream(d)
    cfg = _cfg(oracle, d, f"{variant}_cfg")
    seed = int(d["seed"])
    for tag, stream, delta in (("fine", 2, 0), ("coarse", 2, 2), ("lookup", 3, 0)):
        k = oracle.stream_keys(vs, cfg, seed, stream, delta)
        for f in ("qx", "qy", "qz", "level", "aux", "index", "fingerprint", "jittered"):
            assert np.array_equal(getattr(k, f), d[f"{variant}_{tag}_{f}"]), (tag, f)


def _assert_table(t, d, prefix):
    for f in TABLE_FIELDS:
        assert np.array_equal(getattr(t, f), d[f"{prefix}{f}"]), (prefix, f)


@pytest.mark.parametrize("mode", ["fixed", "float"])
@pytest.mark.parametrize("fixture", ["frame_cornell128.npz", "frame_box4.npz"])
def test_frame_replay(oracle, fixture, mode):
    d = load_golden(fixture)
    vs = golden_stream(d)
    cfg = _cfg(oracle, d, f"{mode}_cfg")
    state = oracle.State.from_config(cfg)
    img, src, chosen, stats = oracle.filter_frame(vs, cfg, state, 0, int(d["seed"]),
                                                  int(d["spp"]), d["base"])
    _assert_table(state.fine, d, f"{mode}_fine_")
    _assert_table(state.coarse, d, f"{mode}_coarse_")
    assert np.array_equal(src, d[f"{mode}_source"])
    assert np.array_equal(chosen, d[f"{mode}_chosen"])
    assert np.array_equal(img, d[f"{mode}_image"])
    lines = str(d[f"{mode}_stats"]).splitlines()
    want = dict(l.split("=", 1) for l in lines)
    assert int(want["probe_failures"]) == stats["probe_failures"]
    assert int(want["collisions"]) == stats["collisions"]


@pytest.mark.parametrize("mode", ["integrate", "filter"])
def test_temporal_corridor_replay(oracle, mode):
    d = load_golden("temporal_corridor.npz")
    cfg = _cfg(oracle, d, f"{mode}_cfg")
    state = oracle.State.from_config(cfg)
    for f in range(int(d["frames"])):
        vs = golden_stream(d, f"f{f}_v_")
        img, src, chosen, _ = oracle.filter_frame(vs, cfg, state, f, int(d[f"f{f}_seed"]), 1,
                                                  d[f"f{f}_base"])
        p = f"{mode}_f{f}_"
        _assert_table(state.fine, d, f"{p}fine_")
        _assert_table(state.coarse, d, f"{p}coarse_")
        assert state.fine.horizon_clears == int(d[f"{p}fine_horizon_clears"])
        assert state.fine.evictions == len(d[f"{p}fine_events"])
        assert np.array_equal(src, d[f"{p}source"])
        assert np.array_equal(img, d[f"{p}image"])


@pytest.mark.parametrize("sm", ["fixed", "float"])
def test_effective_and_begin_frame(oracle, sm):
    d = load_golden("hybrid_table.npz")
    cfg = _cfg(oracle, d, f"{sm}_cfg")
    for f in range(4):
        t = oracle.Table.from_config(cfg)
        for k, v in golden_table(d, f"{sm}_f{f}_pre_").items():
            getattr(t, k)[...] = v
        for mode in ("integrate", "filter", "hybrid"):
            es, ec = t.effective(mode, 0.7, 0.5)
            assert np.array_equal(es, d[f"{sm}_f{f}_eff_{mode}_sum"])
            assert np.array_equal(ec, d[f"{sm}_f{f}_eff_{mode}_cnt"])
    for mode in ("integrate", "filter", "hybrid"):
        t = oracle.Table.from_config(cfg)
        for k, v in golden_table(d, f"{sm}_f3_pre_").items():
            getattr(t, k)[...] = v
        c = oracle.Config(**{**cfg.__dict__, "temporal_mode": mode, "ema_alpha": 0.7})
        t.begin_frame(5, c)
        _assert_table(t, d, f"{sm}_post_{mode}_")


def test_key_stages(oracle):
    """The oracle's per-stage restatements against the reference's vectorised helpers
    (src/keys.py:245-300) on random and edge-case rows (stages.npz)."""
    d = load_golden("stages.npz")
    cfg = _cfg(oracle, d, "cfg")
    lv = oracle.lod(d["camera_distance"], cfg)
    assert np.array_equal(lv, d["levels"])
    t1, t2 = oracle.tangent_frame(d["normal"])
    assert np.array_equal(t1, d["t1"], equal_nan=True)
    assert np.array_equal(t2, d["t2"], equal_nan=True)
    u, v = oracle.disc(d["u1"], d["u2"])
    got = oracle.jitter(d["position"], d["normal"], lv, u, v, cfg)
    assert np.array_equal(got, d["jittered"], equal_nan=True)
    for b in (1, 2, 6, 8, 16, 64):
        assert np.array_equal(oracle.octa_bins(d["normal"], b), d[f"bins_{b}"])
    assert np.array_equal(oracle.aux_word(d["normal"], d["omega_r"], d["layer_id"], cfg), d["aux"])
    cfg2 = _cfg(oracle, d, "cfg_nfp")
    assert np.array_equal(oracle.aux_word(d["normal"], d["omega_r"], d["layer_id"], cfg2),
                          d["aux_nfp"])


@pytest.mark.parametrize("name", ["aux", "delta3", "nfp", "nojit", "probe2", "single", "thr1",
                                  "thr64"])
def test_frame_variants_replay(oracle, name):
    """The oracle frame under each key / ladder option (frame_variants.npz)."""
    d = load_golden("frame_variants.npz")
    vs = golden_stream(d)
    cfg = _cfg(oracle, d, f"{name}_cfg")
    state = oracle.State.from_config(cfg)
    img, src, chosen, stats = oracle.filter_frame(vs, cfg, state, 0, int(d["seed"]),
                                                  int(d["spp"]), d["base"])
    _assert_table(state.fine, d, f"{name}_fine_")
    if state.coarse is not None:
        _assert_table(state.coarse, d, f"{name}_coarse_")
    assert np.array_equal(src, d[f"{name}_source"])
    assert np.array_equal(chosen, d[f"{name}_chosen"])
    assert np.array_equal(img, d[f"{name}_image"])
    want = dict(l.split("=", 1) for l in str(d[f"{name}_stats"]).splitlines())
    assert int(want["probe_failures"]) == stats["probe_failures"]
    assert int(want["collisions"]) == stats["collisions"]
