"""Output formats and keyed temporal helpers against the reference's own outputs
(tests/golden/formats.npz, make_golden.py gen_formats): tone map / PPM bytes
(src/images.py), blend / temporal_difference / migrate_resolution (src/temporal.py),
and -- on the GPU -- VoxelTable.export_csv / dump bytes (src/table.py:314-334)."""

import numpy as np
import pytest

from conftest import golden_table, load_golden


def test_tonemap_and_ppm_bytes(tmp_path):
    from paper_1902_05942_b200.images import read_ppm, tonemap, write_ppm
    d = load_golden("formats.npz")
    assert np.array_equal(tonemap(d["img"]), d["tonemap"])
    write_ppm(tmp_path / "a.ppm", d["img"])
    raw = np.frombuffer((tmp_path / "a.ppm").read_bytes(), np.uint8)
    assert np.array_equal(raw, d["ppm"])
    assert np.array_equal(read_ppm(tmp_path / "a.ppm"), d["tonemap"])
    with pytest.raises(ValueError):
        write_ppm(tmp_path / "b.ppm", np.zeros((4, 4)))


def test_blend_and_temporal_difference():
    from paper_1902_05942_b200.temporal import blend, temporal_difference
    d = load_golden("formats.npz")
    rows = []
    for mode in ("integrate", "filter", "hybrid"):
        for (no, nn, dl) in ((0, 3, 0.0), (5, 0, 0.1), (4, 2, 0.3), (7, 5, 0.9)):
            m, n = blend([0.1, 0.2, 0.3], no, [0.5, 0.25, 0.0], nn, mode, dl)
            rows.append(list(m) + [n])
    assert np.array_equal(np.array(rows), d["blend"])
    got = [temporal_difference([0.1, 0.2, 0.3], [0.2, 0.1, 0.35]),
           temporal_difference([0, 0, 0], [1e-5, 0, 0])]
    assert np.array_equal(np.array(got), d["tdiff"])
    with pytest.raises(ValueError):
        blend([0, 0, 0], 0, [0, 0, 0], 0, "integrate")


def test_migrate_resolution():
    from paper_1902_05942_b200.keys import CellKey
    from paper_1902_05942_b200.temporal import migrate_resolution
    d = load_golden("formats.npz")
    cells = {CellKey(3, -2, 5, 4, 7): (np.array([6.0, 3.0, 1.5]), 6),
             CellKey(2, -2, 5, 4, 7): (np.array([1.0, 1.0, 1.0]), 2),
             CellKey(1, 1, 1, 3, 0): (np.array([2.0, 2.0, 2.0]), 4)}
    for name, (lo, ln, fixed) in {"up": (4, 5, False), "down": (4, 3, False),
                                  "downfix": (4, 2, True)}.items():
        mig = migrate_resolution({k: (np.floor(v * 65536).astype(np.int64) if fixed else v, c)
                                  for k, (v, c) in cells.items()}, lo, ln, 0.25, fixed)
        got = np.array(sorted([k.qx, k.qy, k.qz, k.level, k.aux, c] + [float(x) for x in v]
                              for k, (v, c) in mig.items()))
        assert np.array_equal(got, d[f"mig_{name}"]), name


@pytest.mark.gpu
def test_export_csv_and_dump_bytes(gpu, tmp_path):
    d = load_golden("formats.npz")
    t = gpu.VoxelTable(64, sum_mode="fixed")
    t.load_state(golden_table(d, "csvtab_"))
    t.export_csv(tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text() == str(d["csv"])
    t.dump(tmp_path / "t.bin")
    assert np.array_equal(np.frombuffer((tmp_path / "t.bin").read_bytes(), np.uint8), d["dump"])


class _Desc:
    def __init__(self, vs, i):
        for f in ("position", "normal", "omega_r", "contribution", "throughput"):
            setattr(self, f, getattr(vs, f)[i])
        self.pixel, self.sample = int(vs.pixel[i]), int(vs.sample[i])
        self.layer_id, self.camera_distance = int(vs.layer_id[i]), float(vs.camera_distance[i])


_CFGS = {"default": dict(capacity=1024, footprint_scale=0.002),
         "aux": dict(capacity=1024, footprint_scale=0.002, include_incident_angle=True,
                     include_layer=True)}


@pytest.mark.parametrize("name", list(_CFGS))
def test_scalar_key_path(name):
    """make_cell_key / level_of_detail / jitter_position (src/keys.py:100-240)."""
    from conftest import golden_stream
    from paper_1902_05942_b200.keys import FilterConfig
    from paper_1902_05942_b200.scalar import jitter_position, level_of_detail, make_cell_key
    d = load_golden("formats.npz")
    vs = golden_stream(d, "part_v_")
    cfg = FilterConfig(**_CFGS[name])
    draws = d[f"scalar_{name}_draws"]
    keys = [make_cell_key(_Desc(vs, i), cfg, draws[i], dl) for i in range(len(vs.pixel))
            for dl in (0, 2)]
    got = np.array([[k.qx, k.qy, k.qz, k.level, k.aux] for k in keys])
    assert np.array_equal(got, d[f"scalar_{name}_keys"])
    assert np.array_equal(np.array([level_of_detail(float(x), cfg) for x in vs.camera_distance]),
                          d[f"scalar_{name}_lod"])
    jit = np.array([jitter_position(vs.position[i], vs.normal[i], 3, draws[i], cfg)
                    for i in range(len(vs.pixel))])
    assert np.array_equal(jit, d[f"scalar_{name}_jit"])


@pytest.mark.parametrize("name", list(_CFGS))
@pytest.mark.parametrize("sm", ["fixed", "float"])
def test_brute_partition_csv(tmp_path, name, sm):
    """brute_voxel_average + VoxelPartition.to_csv + neighborhood_mean (src/oracle.py)."""
    from conftest import golden_stream
    from paper_1902_05942_b200.keys import FilterConfig
    from paper_1902_05942_b200.partition import brute_voxel_average, neighborhood_mean
    d = load_golden("formats.npz")
    vs = golden_stream(d, "part_v_")
    part = brute_voxel_average(vs, FilterConfig(**_CFGS[name]), d[f"part_{name}_jittered"], sm)
    part.to_csv(tmp_path / "p.csv")
    assert (tmp_path / "p.csv").read_text() == str(d[f"part_{name}_{sm}_csv"])
    some = sorted(part.cells)[::7]
    assert np.array_equal(np.array([neighborhood_mean(part, k) for k in some]),
                          d[f"part_{name}_{sm}_nbr"])


def test_ball_average_and_mse():
    from conftest import golden_stream
    from paper_1902_05942_b200.partition import ball_average, image_mse
    d = load_golden("formats.npz")
    vs = golden_stream(d, "part_v_")
    got = np.array([ball_average(vs, vs.position[5], 1.5),
                    ball_average(vs, vs.position[9], 0.8,
                                 lambda c, p: 1.0 / (1.0 + float(((p - c) ** 2).sum())))])
    assert np.array_equal(got, d["ball"])
    assert image_mse(d["img"], d["img"] * 0.9) == float(d["mse"])


@pytest.mark.gpu
def test_probe_scan_structured_fingerprints(gpu):
    """normal_in_fingerprint keys share the index hash; probe_scan finds every normal
    variant of a voxel by the fingerprint's spatial bits (src/table.py:186-203)."""
    from paper_1902_05942_b200.scalar import fingerprint_spatial_bits
    d = load_golden("formats.npz")
    t = gpu.VoxelTable(256, sum_mode="fixed", probe_limit=8, ordered=True)
    t.accumulate_batch(d["scan_idx"], d["scan_fp"], d["scan_vals"], 0)
    h = gpu.hashes(gpu.CellKey(4, -3, 9, 2, 0), 0)
    assert h.index == int(d["scan_idx"][0]) and h.fingerprint == int(d["scan_fp"][0])
    sp = fingerprint_spatial_bits(h.fingerprint)
    res = t.probe_scan(h, lambda fp: fingerprint_spatial_bits(fp) == sp)
    assert np.array_equal(np.array([c for _, c in res]), d["scan_counts"])
    assert np.array_equal(np.array([np.asarray(m) for m, _ in res]), d["scan_means"])
