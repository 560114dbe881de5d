"""bench.py's reference arm (CPU): it must run the unmodified reference (baseline/_ref)
on input traced by the reference's own tracer, without importing this repo's package
or mapping its library (the arm's input came from libpf_b200.so)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "pathfilter"))


def test_reference_scene_text_matches_package():
    sys.path.insert(0, ROOT)
    import bench
    from paper_1902_05942_b200.scene import CLOSED_BOX
    assert bench.REF_CLOSED_BOX == CLOSED_BOX


@pytest.mark.skipif(not HAVE_REF, reason="baseline/_ref (reference install) absent")
def test_reference_arm_is_independent_of_the_repo_library():
    code = """
import json, sys
sys.path.insert(0, %r)
import bench
ref = bench.reference_module()
sc, vs, base = bench.reference_stream(ref, 48, 27, 2, 2)
cfg = bench.reference_config(ref, sc, "integrate")
st = ref.FrameState.from_config(cfg)
t = [bench.reference_frame(ref, vs, base, cfg, st, f, 2) for f in range(2)]
mods = [m for m in sys.modules if m.startswith("paper_1902_05942_b200")]
libs = sorted(bench._loaded_libs())
print(json.dumps({"n": len(vs), "mods": mods, "libs": libs, "backend": ref.BACKEND,
                  "cap": cfg.capacity, "fs": cfg.footprint_scale}))
""" % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["mods"] == []
    assert not any("libpf_b200" in p for p in d["libs"])
    assert d["backend"] == "native"
    assert d["cap"] == 1 << (2 * 48 * 27 - 1).bit_length()
    assert d["n"] > 48 * 27
    # same camera footprint as the b200 arm's config
    sys.path.insert(0, ROOT)
    from paper_1902_05942_b200.streams import camera_footprint
    assert d["fs"] == camera_footprint(27)


def test_gpus_flag_starts_that_many_ranks():
    """`bench.py --gpus 2` without a launcher re-executes itself under torchrun (gloo on
    CPU here) and rank 0 reports the world it ran in."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_reduced"] == 2


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode != 0
    assert "refusing" in out.stderr


def test_table_bench_point_lines():
    """paper_1902_05942_b200.bench mirrors src/bench.py's BenchPoint / spread."""
    from paper_1902_05942_b200.bench import BenchPoint, spread
    a = BenchPoint("b200", 100_000, 131072, 1e-4, 2e-5, 1.5e-5)
    b = BenchPoint("b200", 1_000_000, 1 << 20, 4e-4, 1e-4, 5e-5)
    assert a.line().startswith("backend=b200 n=100000 capacity=131072 accumulate_s=0.0001")
    assert "per_vertex_ns=1.2" in a.line() and "device_per_vertex_ns=0.150" in a.line()
    assert abs(spread([a, b]) - 1.2 / 0.5) < 1e-9
    assert abs(spread([a, b], device=True) - 0.15 / 0.05) < 1e-9


def test_occupied_list_key_invalidation():
    """pipeline._occ_key changes on every C-call view of a table (c_table) and on any
    in-place tensor write, so the occupied-slot lists are only reused untouched."""
    import types

    import torch

    from paper_1902_05942_b200.pipeline import _occ_key, _table_key

    def fake():
        t = types.SimpleNamespace(tags=torch.zeros(8, dtype=torch.int64),
                                  counts=torch.zeros(8, dtype=torch.int64),
                                  _sums=torch.zeros(3, 8, dtype=torch.int64),
                                  _cold=torch.zeros(8, 8, dtype=torch.int64))
        return t
    fine, coarse = fake(), fake()
    state = types.SimpleNamespace(fine=fine, coarse=coarse)
    k0 = _occ_key(state)
    assert _occ_key(state) == k0
    fine.__dict__["_c_calls"] = 1          # what VoxelTable.c_table() does
    k1 = _occ_key(state)
    assert k1 != k0
    coarse._cold[3, 2] = 5                 # e.g. set_deltas / a user write
    assert _occ_key(state) != k1
    k2 = _occ_key(state)
    fine._sums.t()[2] = 1                  # a write through a view bumps the base
    assert _occ_key(state) != k2
    assert _table_key(fine)[0] == fine.tags.data_ptr()
    state.coarse = None
    assert _occ_key(state)[1] is None
