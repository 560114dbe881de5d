"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where the reference imports), never on the GPU box:

    PF_REFERENCE=baseline/_ref python tests/golden/make_golden.py

PF_REFERENCE points at a directory containing the reference package `pathfilter`
(the contract's `pip install --target baseline/_ref` of /root/reference/pkg, or a
`setup.py build_ext --inplace` copy's src/).  Every array here is produced by the
reference's own code path (render_frame / accumulate_phase / resolve_phase /
VoxelTable / make_key_arrays); nothing is computed by this repo.
"""

from __future__ import annotations

import json
import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PF_REFERENCE", os.path.join(HERE, "..", "..", "baseline", "_ref"))
sys.path.insert(0, os.path.abspath(REF))

import pathfilter as pf  # noqa: E402
from pathfilter import rng as prng  # noqa: E402
from pathfilter.keys import FilterConfig, hash_arrays, make_key_arrays  # noqa: E402
from pathfilter.pipeline import FrameState, _jitter_draws, accumulate_phase, render_frame, \
    resolve_phase  # noqa: E402
from pathfilter.scene import parse_scene  # noqa: E402
from pathfilter.tracer import TraceOptions, VertexStream, trace  # noqa: E402

assert pf.BACKEND == "native", "build the reference's Cython extension first"

STREAM_FIELDS = ("position", "normal", "omega_r", "contribution", "throughput", "pixel",
                 "sample", "layer_id", "camera_distance")
TABLE_FIELDS = ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas")

CLOSED_BOX = """camera 2.75 2.75 0.6  2.75 2.75 5.5  0 1 0  1.2 {w} {h}
material white 0.73 0.73 0.73
material red 0.65 0.05 0.05
material green 0.12 0.45 0.15
material lamp 0 0 0
quad 0 0 0  0 0 5.5  5.5 0 5.5  5.5 0 0  white
quad 0 5.5 0  5.5 5.5 0  5.5 5.5 5.5  0 5.5 5.5  white
quad 0 0 5.5  0 5.5 5.5  5.5 5.5 5.5  5.5 0 5.5  white
quad 0 0 0  0 5.5 0  0 5.5 5.5  0 0 5.5  red
quad 5.5 0 0  5.5 0 5.5  5.5 5.5 5.5  5.5 5.5 0  green
quad 0 0 0  5.5 0 0  5.5 5.5 0  0 5.5 0  white
quad 1.925 5.49 1.925  3.575 5.49 1.925  3.575 5.49 3.575  1.925 5.49 3.575  lamp emit 17 13 6
"""


def cfg_dict(cfg: FilterConfig) -> str:
    return json.dumps({k: getattr(cfg, k) for k in cfg.__dataclass_fields__})


def put_stream(out: dict, prefix: str, vs: VertexStream):
    for f in STREAM_FIELDS:
        out[f"{prefix}{f}"] = np.ascontiguousarray(getattr(vs, f))


def put_table(out: dict, prefix: str, t):
    for f in TABLE_FIELDS:
        out[f"{prefix}{f}"] = getattr(t, f).copy()
    out[f"{prefix}horizon_clears"] = np.int64(t.horizon_clears)
    ev = t.eviction_events
    out[f"{prefix}events"] = np.array([[e.frame, e.slot, e.victim_age, e.victim_last_touch]
                                       for e in ev], np.int64).reshape(-1, 4)


def put_keys(out: dict, prefix: str, k):
    for f in ("qx", "qy", "qz", "level", "aux", "index", "fingerprint", "jittered"):
        out[f"{prefix}{f}"] = np.ascontiguousarray(getattr(k, f))


def next_pow2(n: int) -> int:
    return 1 << (int(n) - 1).bit_length()


def save(name: str, out: dict):
    out["meta"] = np.array(json.dumps({
        "generator": "tests/golden/make_golden.py", "reference": "pathfilter " + pf.__version__,
        "backend": pf.BACKEND, "numpy": np.__version__, "python": platform.python_version(),
        "libc": " ".join(platform.libc_ver())}))
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **out)
    print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB")


def random_stream(n, seed, n_keys=None, spread=100.0):
    """The reference conftest.random_stream recipe (pkg/tests/conftest.py:28-46),
    plus random layers and exit directions so aux options are exercised."""
    r = np.random.default_rng(seed)
    n_keys = n_keys or max(4, n // 8)
    pts = r.uniform(-spread, spread, (n_keys, 3))
    pick = r.integers(0, n_keys, n)
    normals = r.normal(size=(n, 3))
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    om = r.normal(size=(n, 3))
    om /= np.linalg.norm(om, axis=1, keepdims=True)
    return VertexStream(position=pts[pick], normal=normals, omega_r=om,
                        contribution=r.uniform(0.0, 4.0, (n, 3)), throughput=np.ones((n, 3)),
                        pixel=r.integers(0, 4096, n), sample=r.integers(0, 3, n),
                        layer_id=r.integers(0, 3, n), camera_distance=r.uniform(1.0, 50.0, n))


def gen_rng_hash():
    out = {}
    ids = np.concatenate([np.arange(64, dtype=np.uint64),
                          np.random.default_rng(3).integers(0, 2**63, 192).astype(np.uint64)
                          * np.uint64(2) + np.uint64(1)])
    seeds = [0, 1, 999, 2**63 + 12345, 2**64 - 1]
    for si, seed in enumerate(seeds):
        for stream in (1, 2, 3):
            for dim in (0, 1):
                out[f"draw_u64_{si}_{stream}_{dim}"] = prng.draw_u64_array(seed, stream, ids, 0, dim)
                out[f"draw_unit_{si}_{stream}_{dim}"] = prng.draw_unit_array(seed, stream, ids, 0, dim)
    out["draw_ids"] = ids
    out["draw_seeds"] = np.array(seeds, dtype=np.uint64)
    r = np.random.default_rng(11)
    n = 4096
    q = r.integers(-2**40, 2**40, (n, 3))
    q[:8] = [[0, 0, 0], [1, 0, 0], [-1, 2, -3], [6, -3, 1], [123456, -654321, 42], [0, 0, 0],
             [5, 5, 5], [-1099511627776, 1099511627776, -7]]
    lvl = r.integers(0, 32, n)
    lvl[:8] = [0, 0, 0, 0, 7, 31, 3, 12]
    aux = r.integers(0, 2**32, n).astype(np.uint64)
    aux[:8] = [0, 0, 0, 0, 0, 0, 16909060, 63]
    idx, fp = hash_arrays(q[:, 0], q[:, 1], q[:, 2], lvl, aux)
    bins = r.integers(0, 64, n).astype(np.uint32)
    idx2, fp2 = hash_arrays(q[:, 0], q[:, 1], q[:, 2], lvl, aux, bins)
    out.update(hq=q, hlevel=lvl, haux=aux, hindex=idx, hfp=fp, hbins=bins, hindex_b=idx2,
               hfp_b=fp2)
    save("rng_hash.npz", out)


def gen_keys_random():
    out = {}
    vs = random_stream(3000, seed=7)
    put_stream(out, "v_", vs)
    variants = {
        "default": FilterConfig(base_voxel=0.02, footprint_scale=0.003),
        "aux": FilterConfig(base_voxel=0.02, footprint_scale=0.003, include_incident_angle=True,
                            include_layer=True, normal_bins=6),
        "nfp": FilterConfig(base_voxel=0.05, footprint_scale=0.001, normal_in_fingerprint=True),
        "nojit": FilterConfig(base_voxel=0.02, footprint_scale=0.003, jitter=False,
                              include_normal=False),
    }
    seed = 4242
    for name, cfg in variants.items():
        out[f"{name}_cfg"] = np.array(cfg_dict(cfg))
        for tag, stream, delta in (("fine", 2, 0), ("coarse", 2, 2), ("lookup", 3, 0)):
            u1 = u2 = None
            if cfg.jitter:
                u1, u2 = _jitter_draws(stream, vs, seed)
                out[f"{name}_{tag}_u1"] = u1
                out[f"{name}_{tag}_u2"] = u2
            k = make_key_arrays(vs.position, vs.normal, vs.omega_r, vs.layer_id,
                                vs.camera_distance, cfg, u1, u2, delta)
            put_keys(out, f"{name}_{tag}_", k)
    out["seed"] = np.uint64(seed)
    save("keys_random.npz", out)


def frame_outputs(out, prefix, state, fine_keys, coarse_keys, image, report, stats):
    put_table(out, f"{prefix}fine_", state.fine)
    if state.coarse is not None:
        put_table(out, f"{prefix}coarse_", state.coarse)
    put_keys(out, f"{prefix}fk_", fine_keys)
    if coarse_keys is not None:
        put_keys(out, f"{prefix}ck_", coarse_keys)
    out[f"{prefix}image"] = image
    out[f"{prefix}source"] = report.source
    out[f"{prefix}chosen"] = report.means
    out[f"{prefix}stats"] = np.array("\n".join(l for l in stats.lines() if not l.startswith("time_")))


def gen_frame_cornell():
    out = {}
    scene = pf.cornell_box(128, 128)
    for mode in ("fixed", "float"):
        cfg = FilterConfig(capacity=next_pow2(2 * 128 * 128), sum_mode=mode)
        cfg_f = cfg.for_camera(scene.camera.fov, scene.camera.height)
        state = FrameState.from_config(cfg_f)
        res = render_frame(scene, cfg, state, spp=1, seed=1, threads=1)
        if mode == "fixed":
            put_stream(out, "v_", res.trace_result.vertices)
            out["base"] = res.trace_result.base_image
        out[f"{mode}_cfg"] = np.array(cfg_dict(cfg_f))
        frame_outputs(out, f"{mode}_", state, res.fine_keys, res.coarse_keys, res.filtered,
                      res.report, res.stats)
    out["seed"] = np.uint64(1)
    out["spp"] = np.int64(1)
    save("frame_cornell128.npz", out)


def box_stream(w, h, seed=1):
    scene = parse_scene(CLOSED_BOX.format(w=w, h=h))
    parts, base = [], None
    for k in range(1, 5):
        tr = trace(scene, spp=1, seed=seed, options=TraceOptions(select_k=k, rr_start=9), threads=1)
        vs = tr.vertices
        vs.sample = vs.sample + (k - 1)
        parts.append(vs)
        if k == 1:
            base = tr.base_image
    return scene, VertexStream.concat(parts), base


def gen_frame_box4():
    out = {}
    w, h = 80, 45
    scene, vs, base = box_stream(w, h)
    put_stream(out, "v_", vs)
    out["base"] = base
    seed = 1
    for mode in ("fixed", "float"):
        cfg = FilterConfig(capacity=next_pow2(2 * w * h), sum_mode=mode).for_camera(
            scene.camera.fov, scene.camera.height)
        state = FrameState.from_config(cfg)
        state.fine.begin_frame(0, cfg)
        state.coarse.begin_frame(0, cfg)
        fk, ck, stats = accumulate_phase(vs, cfg, state, 0, seed)
        image, report = resolve_phase(vs, cfg, state, 0, seed, 1, base, fk)
        stats.source_counts = report.counts
        out[f"{mode}_cfg"] = np.array(cfg_dict(cfg))
        frame_outputs(out, f"{mode}_", state, fk, ck, image, report, stats)
    out["seed"] = np.uint64(seed)
    out["spp"] = np.int64(1)
    save("frame_box4.npz", out)


FRAME_VARIANTS = {
    "aux": dict(include_incident_angle=True, include_layer=True, normal_bins=6),
    "nfp": dict(normal_in_fingerprint=True),
    "nojit": dict(jitter=False),
    "single": dict(multi_level=False),
    "thr1": dict(low_count_threshold=1),
    "thr64": dict(low_count_threshold=64),
    "probe2": dict(capacity=512, probe_limit=2),
    "delta3": dict(coarse_delta=3, sum_mode="float"),
}


def gen_frame_variants():
    """One 4-bounce closed-box frame per key / ladder option (the resolve paths the
    default config rarely takes: no coarse table, all-fallback rows, probe failures,
    aux and fingerprint bins in the lookup and pool keys)."""
    out = {}
    w, h = 48, 27
    scene, vs, base = box_stream(w, h, seed=3)
    put_stream(out, "v_", vs)
    out["base"] = base
    seed = 5
    for name, kw in FRAME_VARIANTS.items():
        kw = {"capacity": next_pow2(2 * w * h), **kw}
        cfg = FilterConfig(**kw).for_camera(scene.camera.fov, scene.camera.height)
        state = FrameState.from_config(cfg)
        state.fine.begin_frame(0, cfg)
        if state.coarse is not None:
            state.coarse.begin_frame(0, cfg)
        fk, ck, stats = accumulate_phase(vs, cfg, state, 0, seed)
        image, report = resolve_phase(vs, cfg, state, 0, seed, 1, base, fk)
        stats.source_counts = report.counts
        out[f"{name}_cfg"] = np.array(cfg_dict(cfg))
        frame_outputs(out, f"{name}_", state, fk, ck, image, report, stats)
    out["seed"] = np.uint64(seed)
    out["spp"] = np.int64(1)
    out["variants"] = np.array(sorted(FRAME_VARIANTS))
    save("frame_variants.npz", out)


def gen_temporal():
    """Corridor pan with a 128-slot table: claims, evictions and horizon clears."""
    out = {}
    frames = 10
    scene = pf.scene.corridor(24, 24, frames=frames)
    for mode in ("integrate", "filter"):
        cfg = FilterConfig(capacity=128, probe_limit=4, temporal_mode=mode, evict_horizon=3,
                           evict_min_age=1, sample_cap=24)
        cfg_f = cfg.for_camera(scene.camera.fov, scene.camera.height)
        state = FrameState.from_config(cfg_f)
        out[f"{mode}_cfg"] = np.array(cfg_dict(cfg_f))
        for f in range(frames):
            res = render_frame(scene, cfg, state, spp=1, seed=5, threads=1)
            p = f"{mode}_f{f}_"
            if mode == "integrate":
                put_stream(out, f"f{f}_v_", res.trace_result.vertices)
                out[f"f{f}_base"] = res.trace_result.base_image
                out[f"f{f}_seed"] = np.uint64(state.prev_seed)
            put_table(out, f"{p}fine_", state.fine)
            put_table(out, f"{p}coarse_", state.coarse)
            out[f"{p}image"] = res.filtered
            out[f"{p}source"] = res.report.source
            out[f"{p}chosen"] = res.report.means
    out["frames"] = np.int64(frames)
    save("temporal_corridor.npz", out)


def gen_hybrid():
    """effective()/begin_frame() in hybrid and filter modes with nonzero deltas."""
    from pathfilter.table import VoxelTable
    out = {}
    vs = random_stream(2000, seed=9, n_keys=300, spread=2.0)
    for sm in ("fixed", "float"):
        cfg = FilterConfig(capacity=1024, probe_limit=8, temporal_mode="hybrid", sample_cap=5,
                           sum_mode=sm, base_voxel=0.05, footprint_scale=0.002)
        keys = make_key_arrays(vs.position, vs.normal, vs.omega_r, vs.layer_id,
                               vs.camera_distance, cfg)
        t = VoxelTable.from_config(cfg)
        r = np.random.default_rng(1)
        for f in range(4):
            t.begin_frame(f, cfg)
            part = slice(f * 400, f * 400 + 900)
            t.accumulate_batch(keys.index[part], keys.fingerprint[part], vs.contribution[part], f)
            occ = np.nonzero(t.tags != np.uint64(0xFFFFFFFF00000000))[0]
            t.set_deltas(occ, r.uniform(0.0, 0.8, len(occ)))
            put_table(out, f"{sm}_f{f}_pre_", t)
            for mode in ("integrate", "filter", "hybrid"):
                es, ec = t.effective(mode, 0.7, 0.5)
                out[f"{sm}_f{f}_eff_{mode}_sum"] = es
                out[f"{sm}_f{f}_eff_{mode}_cnt"] = ec
        for mode in ("integrate", "filter", "hybrid"):
            t2 = VoxelTable.from_config(cfg)
            for k in TABLE_FIELDS:
                getattr(t2, k)[...] = out[f"{sm}_f3_pre_{k}"]
            c2 = FilterConfig(**{**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__},
                                 "temporal_mode": mode, "ema_alpha": 0.7})
            t2.begin_frame(5, c2)
            put_table(out, f"{sm}_post_{mode}_", t2)
        out[f"{sm}_cfg"] = np.array(cfg_dict(cfg))
    save("hybrid_table.npz", out)


def put_trace(out: dict, prefix: str, res):
    put_stream(out, f"{prefix}v_", res.vertices)
    out[f"{prefix}image"] = res.image
    out[f"{prefix}base"] = res.base_image
    if res.variance is not None:
        out[f"{prefix}variance"] = res.variance


def gen_tracer():
    """Phase-one fixtures: the reference tracer (src/tracer.py) on every builtin scene
    kind, the benchmark's closed box (select_k = 1..4, rr_start 9), glossy layers,
    motion, RR, NEE off / no pixel jitter, variance, and a reevaluate replay."""
    from pathfilter.scene import load_scene
    from pathfilter.tracer import reevaluate
    out = {}
    box = parse_scene(CLOSED_BOX.format(w=48, h=27))
    for k in range(1, 5):
        put_trace(out, f"box_k{k}_", trace(box, 1, 1, TraceOptions(select_k=k, rr_start=9)))
    put_trace(out, "cornell_", trace(load_scene("cornell", 32, 32), 2, 5, want_variance=True))
    put_trace(out, "glossy_", trace(load_scene("cornell-glossy", 24, 24), 1, 3,
                                    TraceOptions(select_k=2)))
    sweep = load_scene("shadow-sweep", 24, 24).at_frame(3)
    put_trace(out, "sweep_", trace(sweep, 1, 7))
    put_trace(out, "occluded_", trace(load_scene("occluded", 8, 8), 1, 2))
    corr = load_scene("corridor", 20, 16).at_frame(5)
    put_trace(out, "corridor_", trace(corr, 1, 9, TraceOptions(nee=False, pixel_jitter=False,
                                                                max_depth=5)))
    cb = load_scene("cornell", 32, 32)
    ids = (np.arange(0, 2048, 7, dtype=np.uint64) % np.uint64(1024)) | \
        ((np.arange(0, 2048, 7, dtype=np.uint64) // np.uint64(1024)) << np.uint64(32))
    out["reeval_ids"] = ids
    put_stream(out, "reeval_v_", reevaluate(cb, 5, 2, ids))
    for name, sc in (("box", box), ("cornell", cb), ("glossy", load_scene("cornell-glossy", 24, 24)),
                     ("sweep3", sweep), ("occluded", load_scene("occluded", 8, 8)),
                     ("corridor5", corr)):
        for f in ("v0", "e1", "e2", "normal", "area", "material_id", "emission"):
            out[f"scene_{name}_{f}"] = getattr(sc, f)
        out[f"scene_{name}_basis"] = np.stack(sc.camera.basis())
    save("tracer.npz", out)


def gen_render():
    """render_frame sequences (src/pipeline.py:321-380): trace + temporal update +
    accumulate (+ hybrid replay) + resolve, per temporal mode."""
    from pathfilter.pipeline import run_sequence
    from pathfilter.scene import load_scene
    out = {}
    runs = {
        "integrate": ("cornell", 24, 24, 2, dict()),
        "filter": ("corridor", 20, 16, 4, dict(temporal_mode="filter")),
        "hybrid": ("shadow-sweep", 24, 24, 4, dict(temporal_mode="hybrid",
                                                   reevaluate_fraction=0.25)),
    }
    for name, (scene_name, w, h, frames, kw) in runs.items():
        sc = load_scene(scene_name, w, h)
        cfg = FilterConfig(capacity=next_pow2(2 * w * h), **kw)
        res = run_sequence(sc, cfg, 1, 13, frames=frames)
        out[f"{name}_cfg"] = np.array(cfg_dict(cfg))
        out[f"{name}_meta"] = np.array(json.dumps([scene_name, w, h, frames]))
        for f, r in enumerate(res):
            out[f"{name}_f{f}_filtered"] = r.filtered
            out[f"{name}_f{f}_unfiltered"] = r.unfiltered
            out[f"{name}_f{f}_source"] = r.report.source
            out[f"{name}_f{f}_stats"] = np.array("\n".join(r.stats.lines()))
    save("render.npz", out)


def gen_formats():
    """Output formats and the keyed temporal helpers: tonemap / PPM
    bytes (src/images.py), VoxelTable.export_csv / dump bytes, blend /
    temporal_difference / migrate_resolution (src/temporal.py)."""
    import io
    import tempfile
    from pathfilter.images import tonemap, write_ppm
    from pathfilter.keys import CellKey
    from pathfilter.table import VoxelTable
    from pathfilter.temporal import blend, migrate_resolution, temporal_difference
    r = np.random.default_rng(5)
    out = {}
    img = r.uniform(-0.2, 1.4, (7, 9, 3))
    out["img"] = img
    out["tonemap"] = tonemap(img)
    with tempfile.TemporaryDirectory() as td:
        write_ppm(os.path.join(td, "a.ppm"), img)
        out["ppm"] = np.frombuffer(open(os.path.join(td, "a.ppm"), "rb").read(), np.uint8)
        t = VoxelTable(64, sum_mode="fixed")
        vs = random_stream(200, 3, n_keys=20, spread=2.0)
        k = make_key_arrays(vs.position, vs.normal, vs.omega_r, vs.layer_id, vs.camera_distance,
                            FilterConfig(capacity=64), None, None, 0)
        t.accumulate_batch(k.index, k.fingerprint, vs.contribution, 0)
        put_table(out, "csvtab_", t)
        t.export_csv(os.path.join(td, "t.csv"))
        out["csv"] = np.array(open(os.path.join(td, "t.csv")).read())
        t.dump(os.path.join(td, "t.bin"))
        out["dump"] = np.frombuffer(open(os.path.join(td, "t.bin"), "rb").read(), np.uint8)
    rows = []
    for mode in ("integrate", "filter", "hybrid"):
        for (no, nn, dl) in ((0, 3, 0.0), (5, 0, 0.1), (4, 2, 0.3), (7, 5, 0.9)):
            m, n = blend([0.1, 0.2, 0.3], no, [0.5, 0.25, 0.0], nn, mode, dl)
            rows.append(list(m) + [n])
    out["blend"] = np.array(rows)
    out["tdiff"] = np.array([temporal_difference([0.1, 0.2, 0.3], [0.2, 0.1, 0.35]),
                             temporal_difference([0, 0, 0], [1e-5, 0, 0])])
    cells = {CellKey(3, -2, 5, 4, 7): (np.array([6.0, 3.0, 1.5]), 6),
             CellKey(2, -2, 5, 4, 7): (np.array([1.0, 1.0, 1.0]), 2),
             CellKey(1, 1, 1, 3, 0): (np.array([2.0, 2.0, 2.0]), 4)}
    for name, (lo, ln, fixed) in {"up": (4, 5, False), "down": (4, 3, False),
                                  "downfix": (4, 2, True)}.items():
        mig = migrate_resolution({k: (np.floor(v * 65536).astype(np.int64) if fixed else v, c)
                                  for k, (v, c) in cells.items()}, lo, ln, 0.25, fixed)
        out[f"mig_{name}"] = np.array(sorted(
            [k.qx, k.qy, k.qz, k.level, k.aux, c] + [float(x) for x in v]
            for k, (v, c) in mig.items()))
    # scalar key path + brute-force partition utilities (src/keys.py:100-240, src/oracle.py)
    from pathfilter.keys import jitter_position, level_of_detail, make_cell_key
    from pathfilter.oracle import ball_average, brute_voxel_average, image_mse, \
        neighborhood_mean
    vs = random_stream(300, 11, n_keys=40, spread=3.0)
    cfgs = {"default": FilterConfig(capacity=1024, footprint_scale=0.002),
            "aux": FilterConfig(capacity=1024, footprint_scale=0.002, include_incident_angle=True,
                                include_layer=True)}
    for name, cfg in cfgs.items():
        draws = r.random((len(vs), 2))
        keys = [make_cell_key(vs.descriptor(i), cfg, draws[i], d) for i in range(len(vs))
                for d in (0, 2)]
        out[f"scalar_{name}_draws"] = draws
        out[f"scalar_{name}_keys"] = np.array([[k.qx, k.qy, k.qz, k.level, k.aux] for k in keys])
        out[f"scalar_{name}_lod"] = np.array([level_of_detail(float(d), cfg)
                                              for d in vs.camera_distance])
        out[f"scalar_{name}_jit"] = np.array([jitter_position(vs.position[i], vs.normal[i], 3,
                                                              draws[i], cfg)
                                              for i in range(len(vs))])
        ka = make_key_arrays(vs.position, vs.normal, vs.omega_r, vs.layer_id, vs.camera_distance,
                             cfg, draws[:, 0], draws[:, 1], 0)
        out[f"part_{name}_jittered"] = ka.jittered
        for sm in ("fixed", "float"):
            part = brute_voxel_average(vs, cfg, ka.jittered, sm)
            with tempfile.TemporaryDirectory() as td:
                part.to_csv(os.path.join(td, "p.csv"))
                out[f"part_{name}_{sm}_csv"] = np.array(open(os.path.join(td, "p.csv")).read())
            some = sorted(part.cells)[::7]
            out[f"part_{name}_{sm}_nbr"] = np.array([neighborhood_mean(part, k) for k in some])
    put_stream(out, "part_v_", vs)
    out["ball"] = np.array([ball_average(vs, vs.position[5], 1.5),
                            ball_average(vs, vs.position[9], 0.8,
                                         lambda c, p: 1.0 / (1.0 + float(((p - c) ** 2).sum())))])
    out["mse"] = np.array(image_mse(img, img * 0.9))
    # probe_scan over structured fingerprints (normal_in_fingerprint, src/table.py:186-203)
    from pathfilter.keys import fingerprint_spatial_bits, hashes as ref_hashes
    t = VoxelTable(256, sum_mode="fixed", probe_limit=8)
    key = CellKey(4, -3, 9, 2, 0)
    idx, fps, vals = [], [], []
    for nb in range(6):
        h = ref_hashes(key, nb)
        idx.append(h.index)
        fps.append(h.fingerprint)
        vals.append([0.1 * nb, 0.2, 0.3 + nb])
    other = ref_hashes(CellKey(5, -3, 9, 2, 0), 1)
    idx.append(other.index)
    fps.append(other.fingerprint)
    vals.append([9.0, 9.0, 9.0])
    t.accumulate_batch(np.array(idx, np.uint64), np.array(fps, np.uint32), np.array(vals), 0)
    sp = fingerprint_spatial_bits(ref_hashes(key, 0).fingerprint)
    res = t.probe_scan(ref_hashes(key, 0), lambda fp: fingerprint_spatial_bits(fp) == sp)
    out["scan_idx"], out["scan_fp"] = np.array(idx, np.uint64), np.array(fps, np.uint32)
    out["scan_vals"] = np.array(vals)
    out["scan_means"] = np.array([m for m, _ in res])
    out["scan_counts"] = np.array([c for _, c in res])
    save("formats.npz", out)


def gen_stages():
    """The per-stage vectorised helpers (src/keys.py:245-300) on random and edge-case rows:
    signed zeros, axis normals, the -z hemisphere seam, ratios around 1 and 2^k, huge
    distances, unnormalised normals."""
    from pathfilter.keys import aux_bits_array, jittered_positions, levels_array, \
        normal_bins_array, tangent_basis_array
    out = {}
    r = np.random.default_rng(21)
    n = 6000
    nrm = r.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    edge = np.array([[0, 0, 1], [0, 0, -1], [0, 0, 0.0], [0, 0, -0.0], [1, 0, 0], [-1, 0, 0],
                     [0, 1, 0], [0, -1, 0], [0.6, 0.8, -0.0], [-0.6, 0.8, 0.0],
                     [1e-300, -1e-300, -1], [3.0, -4.0, 12.0], [0.5, 0.5, -0.5],
                     [-0.0, -0.0, -1.0], [1e-17, 1.0, -1e-17], [0, 0, 0]], np.float64)
    nrm[:len(edge)] = edge
    om = r.normal(size=(n, 3))
    om /= np.linalg.norm(om, axis=1, keepdims=True)
    om[:len(edge)] = edge[::-1]
    lay = r.integers(0, 3, n)
    dist = np.exp(r.uniform(np.log(1e-3), np.log(1e7), n))
    cfg = FilterConfig(base_voxel=0.02, footprint_scale=0.003, include_incident_angle=True,
                       include_layer=True, normal_bins=6)
    c_lod = cfg.footprint_scale * cfg.s_pixels / cfg.base_voxel
    ks = np.arange(32)
    near = np.concatenate([2.0 ** ks, np.nextafter(2.0 ** ks, 0), np.nextafter(2.0 ** ks, 3e9)])
    dist[:len(near)] = near / c_lod
    dist[len(near):len(near) + 4] = [0.0, 1e-300, 1e300, 1.0 / c_lod]
    u1 = r.uniform(0.0, 1.0, n)
    u2 = r.uniform(0.0, 1.0, n)
    u1[:4] = [0.0, 1.0, 0.5, np.nextafter(1.0, 0)]
    u2[:4] = [0.0, 0.25, 0.999999999, 0.5]
    pos = r.uniform(-100.0, 100.0, (n, 3))
    lv = levels_array(dist, cfg)
    t1, t2 = tangent_basis_array(nrm)
    out.update(normal=nrm, omega_r=om, layer_id=lay, camera_distance=dist, u1=u1, u2=u2,
               position=pos, cfg=np.array(cfg_dict(cfg)), levels=lv, t1=t1, t2=t2,
               jittered=jittered_positions(pos, nrm, lv, u1, u2, cfg),
               jittered_lv0=jittered_positions(pos, nrm, np.zeros(n, np.int64), u1, u2, cfg),
               aux=aux_bits_array(nrm, om, lay, cfg))
    for b in (1, 2, 6, 8, 16, 64):
        out[f"bins_{b}"] = normal_bins_array(nrm, b)
    cfg2 = FilterConfig(include_normal=True, normal_in_fingerprint=True, include_layer=True)
    out["cfg_nfp"] = np.array(cfg_dict(cfg2))
    out["aux_nfp"] = aux_bits_array(nrm, om, lay, cfg2)
    # keys of vertices whose jittered distance straddles a LOD threshold: distances just
    # below d_k = 2^k / c_lod (within the fine and coarse jitter radii) and around it
    m = 12000
    k = r.integers(1, 24, m)
    rel = np.where(r.uniform(size=m) < 0.5, r.uniform(0.0, 0.004, m), r.uniform(0.0, 0.03, m))
    near = (2.0 ** k / c_lod) * (1.0 - rel)
    near[:64] = np.nextafter(2.0 ** k[:64] / c_lod, 0.0)
    near[64:128] = 2.0 ** k[64:128] / c_lod
    near[128:136] = [0.0, 1e-300, 1e300, np.inf, 31.9 / c_lod, 2.0 ** 31 / c_lod, 1e9, 5e8]
    npos = r.uniform(-100.0, 100.0, (m, 3))
    nn = r.normal(size=(m, 3))
    nn /= np.linalg.norm(nn, axis=1, keepdims=True)
    nl = r.integers(0, 3, m)
    nu1, nu2 = r.uniform(0.0, 1.0, m), r.uniform(0.0, 1.0, m)
    nu1[:512] = 1.0 - r.uniform(0.0, 1e-6, 512)  # the full jitter radius
    out.update(near_position=npos, near_normal=nn, near_layer=nl, near_distance=near,
               near_u1=nu1, near_u2=nu2)
    for delta in (0, 2):
        kk = make_key_arrays(npos, nn, nn, nl, near, cfg, nu1, nu2, delta)
        put_keys(out, f"near{delta}_", kk)
    save("stages.npz", out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "keys", "cornell", "box4", "temporal", "hybrid", "tracer",
                             "render", "formats", "stages", "variants"]
    fns = {"rng": gen_rng_hash, "keys": gen_keys_random, "cornell": gen_frame_cornell,
           "box4": gen_frame_box4, "temporal": gen_temporal, "hybrid": gen_hybrid,
           "tracer": gen_tracer, "render": gen_render, "formats": gen_formats,
           "stages": gen_stages, "variants": gen_frame_variants}
    for w in which:
        fns[w]()
