"""CPU: the scene module (paper_1902_05942_b200/scene.py) builds the reference's scenes
exactly -- triangle arrays, normals, areas, materials, motion and camera bases match
the arrays the reference produced (tests/golden/tracer.npz, make_golden.py gen_tracer)."""

import numpy as np
import pytest

from conftest import load_golden


def _scenes():
    from paper_1902_05942_b200 import scene as S
    return {
        "box": S.closed_box(48, 27),
        "cornell": S.load_scene("cornell", 32, 32),
        "glossy": S.load_scene("cornell-glossy", 24, 24),
        "sweep3": S.load_scene("shadow-sweep", 24, 24).at_frame(3),
        "occluded": S.load_scene("occluded", 8, 8),
        "corridor5": S.load_scene("corridor", 20, 16).at_frame(5),
    }


@pytest.mark.parametrize("name", ["box", "cornell", "glossy", "sweep3", "occluded", "corridor5"])
def test_builtin_scenes_match_reference(name):
    d = load_golden("tracer.npz")
    sc = _scenes()[name]
    for f in ("v0", "e1", "e2", "normal", "area", "material_id", "emission"):
        assert np.array_equal(getattr(sc, f), d[f"scene_{name}_{f}"]), f
    assert np.array_equal(np.stack(sc.camera.basis()), d[f"scene_{name}_basis"])


def test_parse_errors_and_directives():
    from paper_1902_05942_b200.scene import SceneError, parse_scene
    good = """camera 0 0 -5  0 0 0  0 1 0  1.0 4 3
material m 0.5 0.5 0.5 glossy 0.2 10
material lamp 0 0 0
tri 0 0 0  1 0 0  0 1 0  m
quad -1 2 -1  1 2 -1  1 2 1  -1 2 1  lamp emit 1 2 3   # a comment
background 0.1 0.2 0.3
frames 4
move camera 1 0 0
move lights 0 1 0
emission_scale 0.5
"""
    sc = parse_scene(good)
    assert len(sc.v0) == 3 and sc.frames == 4
    assert sc.materials[0].glossy_weight == 0.2 and sc.materials[0].glossy_exponent == 10.0
    assert np.array_equal(sc.background, [0.1, 0.2, 0.3])
    f2 = sc.at_frame(2)
    assert np.array_equal(f2.camera.position, [2.0, 0.0, -5.0])
    assert np.array_equal(f2.v0[1:], sc.v0[1:] + [0.0, 2.0, 0.0])
    assert np.array_equal(f2.emission, sc.emission * 0.25)
    for bad in ("bogus 1 2 3", "camera 1 2 3", "material q 1 1", "material q 2 0 0",
                "tri 0 0 0 1 0 0 0 1 0", "move planet 1 0 0"):
        with pytest.raises(SceneError):
            parse_scene(good + bad + "\n")
    with pytest.raises(SceneError):
        parse_scene("material m 0.5 0.5 0.5\n")  # no camera
