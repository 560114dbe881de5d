"""Output formats and keyed temporal helpers against the reference's own outputs
(tests/golden/formats.npz, make_golden.py gen_formats): tone map / PPM bytes
(src/images.py), migrate_resolution (src/temporal.py, on the device),
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


@pytest.mark.gpu
def test_migrate_resolution(gpu):
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


@pytest.mark.gpu
def test_probe_scan_structured_fingerprints(gpu):
    """normal_in_fingerprint keys share the index hash; probe_scan finds every normal
    variant of a voxel by the fingerprint's spatial bits (src/table.py:186-203)."""
    def fingerprint_spatial_bits(fp):   # src/keys.py:237-240: the bits above the normal bins
        return fp >> 6
    d = load_golden("formats.npz")
    t = gpu.VoxelTable(256, sum_mode="fixed", probe_limit=8, ordered=True)
    t.accumulate_batch(d["scan_idx"], d["scan_fp"], d["scan_vals"], 0)
    h = gpu.hashes(gpu.CellKey(4, -3, 9, 2, 0), 0)
    assert h.index == int(d["scan_idx"][0]) and h.fingerprint == int(d["scan_fp"][0])
    sp = fingerprint_spatial_bits(h.fingerprint)
    res = t.probe_scan(h, lambda fp: fingerprint_spatial_bits(fp) == sp)
    assert np.array_equal(np.array([c for _, c in res]), d["scan_counts"])
    assert np.array_equal(np.array([np.asarray(m) for m, _ in res]), d["scan_means"])


@pytest.mark.gpu
@pytest.mark.parametrize("lo,ln,fixed", [(2, 3, False), (2, 4, True), (3, 1, False),
                                          (3, 2, True), (2, 2, False)])
def test_migrate_resolution_matches_reference_with_collisions(gpu, lo, ln, fixed):
    """Random snapshots whose keys collide after migration (children of one parent,
    pass-through keys equal to a parent or child, in every order) against the
    reference's own migrate_resolution (baseline/_ref, src/temporal.py:107-151): same
    keys in the same dict order, same counts, sums bit for bit."""
    import os
    import sys
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "pathfilter")):
        pytest.skip("baseline/_ref absent")
    sys.path.insert(0, ref)
    from pathfilter.keys import CellKey as RKey
    from pathfilter.temporal import migrate_resolution as ref_migrate
    from paper_1902_05942_b200.keys import CellKey
    from paper_1902_05942_b200.temporal import migrate_resolution
    r = np.random.default_rng(lo * 10 + ln)
    cells_ref, cells = {}, {}
    for _ in range(300):
        q = r.integers(-6, 6, 3)
        lvl = int(r.choice([lo, lo, ln, 5]))
        aux = int(r.integers(0, 2))
        tot = r.uniform(0, 9, 3)
        if fixed:
            tot = np.floor(tot * 65536).astype(np.int64)
        c = int(r.integers(1, 40))
        k = (int(q[0]), int(q[1]), int(q[2]), lvl, aux)
        cells_ref[RKey(*k)] = (tot, c)
        cells[CellKey(*k)] = (tot, c)
    want = ref_migrate(cells_ref, lo, ln, 0.25, fixed)
    got = migrate_resolution(cells, lo, ln, 0.25, fixed)
    kt = lambda k: (k.qx, k.qy, k.qz, k.level, k.aux)  # noqa: E731
    assert [kt(k) for k in got] == [kt(k) for k in want]
    for (kg, (sg, cg)), (kw, (sw, cw)) in zip(got.items(), want.items()):
        assert cg == cw, kg
        assert np.array_equal(np.asarray(sg), np.asarray(sw)), kg
