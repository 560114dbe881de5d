"""Scenes for the on-device path tracer (phase one).

A restatement of the reference scene model (src/scene.py): a triangle soup
with per-triangle material and emission, a pinhole camera, per-frame motion,
the builder, the line-based text format (src/scene.py:359-421) and the builtin
scenes (src/scene.py:198-330), plus the closed box of the benchmark.
Scenes live on the host (a few hundred triangles at most); `device_tables()`
uploads the flat arrays the CUDA tracer indexes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np


class SceneError(ValueError):
    """Invalid scene definition (src/scene.py:17-18)."""


def _vec(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).reshape(3)


@dataclass
class Camera:
    """Pinhole camera; fov is the vertical field of view in radians (src/scene.py:21-44)."""

    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    fov: float
    width: int
    height: int

    def basis(self):
        """(right, up, forward), right-handed, as numpy computes it."""
        fwd = self.look_at - self.position
        length = np.linalg.norm(fwd)
        if length == 0.0:
            raise SceneError("camera position and look_at coincide")
        fwd = fwd / length
        right = np.cross(fwd, self.up)
        rl = np.linalg.norm(right)
        if rl < 1e-12:
            raise SceneError("camera up is parallel to the view direction")
        right = right / rl
        return right, np.cross(right, fwd), fwd


@dataclass
class Material:
    """Diffuse albedo plus an optional Phong glossy lobe (src/scene.py:47-56)."""

    name: str
    albedo: np.ndarray
    glossy_weight: float = 0.0
    glossy_exponent: float = 0.0

    @property
    def diffuse_weight(self) -> float:
        return 1.0 - self.glossy_weight


@dataclass
class Motion:
    """Linear per-frame motion (src/scene.py:59-65)."""

    camera_velocity: np.ndarray | None = None
    light_velocity: np.ndarray | None = None
    emission_scale: float | None = None


@dataclass
class Scene:
    """Triangle arrays (M, 3) with edges e1 = b - a, e2 = c - a (src/scene.py:68-133)."""

    camera: Camera
    materials: list
    v0: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    e1: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    e2: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    normal: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    area: np.ndarray = field(default_factory=lambda: np.zeros(0))
    material_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    emission: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    frames: int = 1
    motion: Motion = field(default_factory=Motion)

    @property
    def light_indices(self) -> np.ndarray:
        return np.nonzero(self.emission.max(axis=1) > 0.0)[0]

    @property
    def max_emission(self) -> float:
        return float(self.emission.max()) if len(self.emission) else 0.0

    def validate(self) -> "Scene":
        cam = self.camera
        problems = []
        if not 0.0 < cam.fov < math.pi:
            problems.append("camera fov must be in (0, pi)")
        if cam.width < 1 or cam.height < 1:
            problems.append("image dimensions must be positive")
        if len(self.v0) == 0:
            problems.append("scene has no geometry")
        elif np.any(self.area <= 1e-14):
            problems.append("degenerate (zero-area) triangle in scene")
        for m in self.materials:
            if np.any(m.albedo < 0.0) or np.any(m.albedo > 1.0):
                problems.append(f"material {m.name!r}: albedo outside [0, 1]")
            if not 0.0 <= m.glossy_weight <= 1.0:
                problems.append(f"material {m.name!r}: glossy weight outside [0, 1]")
        if len(self.v0) and len(self.light_indices) == 0:
            problems.append("scene has no light source")
        if np.any(self.emission < 0.0):
            problems.append("negative emission")
        if problems:
            raise SceneError(problems[0])
        cam.basis()
        return self

    def at_frame(self, frame: int) -> "Scene":
        """The scene at frame `frame` under its motion block."""
        mo = self.motion
        if frame == 0 or (mo.camera_velocity is None and mo.light_velocity is None
                          and mo.emission_scale is None):
            return self
        out = replace(self)
        if mo.camera_velocity is not None:
            shift = mo.camera_velocity * frame
            out.camera = replace(self.camera, position=self.camera.position + shift,
                                 look_at=self.camera.look_at + shift)
        if mo.light_velocity is not None:
            moved = self.v0.copy()
            moved[self.emission.max(axis=1) > 0.0] += mo.light_velocity * frame
            out.v0 = moved
        if mo.emission_scale is not None:
            out.emission = self.emission * (mo.emission_scale ** frame)
        return out

    # -- device view ---------------------------------------------------------------

    def device_tables(self, device=None) -> dict:
        """Flat float64 / int arrays the tracer kernel reads (uploaded once)."""
        import torch
        dev = torch.device(device) if device is not None else torch.device("cuda")

        def t(a, dt=torch.float64):
            return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

        mats = self.materials
        return {
            "v0": t(self.v0), "e1": t(self.e1), "e2": t(self.e2), "normal": t(self.normal),
            "emission": t(self.emission), "area": t(self.area),
            "material_id": t(self.material_id, torch.int32),
            "albedo": t(np.stack([m.albedo for m in mats])),
            "glossy_weight": t(np.array([m.glossy_weight for m in mats])),
            "glossy_exponent": t(np.array([m.glossy_exponent for m in mats])),
            "light_tri": t(self.light_indices.astype(np.int64), torch.int64),
        }


class SceneBuilder:
    """Collects materials and triangles, then freezes a Scene (src/scene.py:136-195)."""

    def __init__(self):
        self.camera: Camera | None = None
        self.materials: list = []
        self._ids: dict = {}
        self._tris: list = []
        self.background = np.zeros(3)
        self.frames = 1
        self.motion = Motion()

    def add_material(self, m: Material) -> int:
        if m.name in self._ids:
            raise SceneError(f"duplicate material {m.name!r}")
        self._ids[m.name] = len(self.materials)
        self.materials.append(m)
        return self._ids[m.name]

    def material_id(self, name: str) -> int:
        try:
            return self._ids[name]
        except KeyError:
            raise SceneError(f"unknown material {name!r}") from None

    def add_triangle(self, a, b, c, material: str, emission=(0.0, 0.0, 0.0)):
        self._tris.append((_vec(a), _vec(b), _vec(c), self.material_id(material), _vec(emission)))

    def add_quad(self, a, b, c, d, material: str, emission=(0.0, 0.0, 0.0)):
        """Quad in winding order as the fan (a, b, c), (a, c, d)."""
        self.add_triangle(a, b, c, material, emission)
        self.add_triangle(a, c, d, material, emission)

    def build(self) -> Scene:
        if self.camera is None:
            raise SceneError("scene has no camera")
        if self._tris:
            a = np.stack([t[0] for t in self._tris])
            e1 = np.stack([t[1] for t in self._tris]) - a
            e2 = np.stack([t[2] for t in self._tris]) - a
            mid = np.array([t[3] for t in self._tris], np.int32)
            em = np.stack([t[4] for t in self._tris])
        else:
            a = e1 = e2 = em = np.zeros((0, 3))
            mid = np.zeros(0, np.int32)
        cr = np.cross(e1, e2)
        length = np.linalg.norm(cr, axis=1)
        with np.errstate(invalid="ignore", divide="ignore"):
            nrm = np.where(length[:, None] > 0, cr / np.maximum(length, 1e-300)[:, None], 0.0)
        return Scene(camera=self.camera, materials=list(self.materials), v0=a, e1=e1, e2=e2,
                     normal=nrm, area=0.5 * length, material_id=mid, emission=em,
                     background=self.background, frames=self.frames,
                     motion=self.motion).validate()


def _box(b: SceneBuilder, s: float, walls: dict):
    """The five/six axis-aligned walls of [0, s]^3 with inward normals."""
    quads = {
        "floor": ((0, 0, 0), (0, 0, s), (s, 0, s), (s, 0, 0)),
        "ceiling": ((0, s, 0), (s, s, 0), (s, s, s), (0, s, s)),
        "back": ((0, 0, s), (0, s, s), (s, s, s), (s, 0, s)),
        "left": ((0, 0, 0), (0, s, 0), (0, s, s), (0, 0, s)),
        "right": ((s, 0, 0), (s, 0, s), (s, s, s), (s, s, 0)),
    }
    for wall, mat in walls.items():
        b.add_quad(*quads[wall], mat)


def cornell_box(width: int = 64, height: int = 64, glossy_back: bool = False) -> Scene:
    """Open-front Cornell box with a ceiling lamp (src/scene.py:198-234)."""
    s = 5.5
    b = SceneBuilder()
    b.camera = Camera(_vec((s / 2, s / 2, -8.0)), _vec((s / 2, s / 2, 0.0)), _vec((0, 1, 0)),
                      2.0 * math.atan((s / 2) / 8.0), width, height)
    for name, rgb in (("white", (0.73, 0.73, 0.73)), ("red", (0.65, 0.05, 0.05)),
                      ("green", (0.12, 0.45, 0.15)), ("lamp", (0.0, 0.0, 0.0))):
        b.add_material(Material(name, _vec(rgb)))
    if glossy_back:
        b.add_material(Material("glossyback", _vec((0.6, 0.6, 0.7)), 0.3, 40.0))
    _box(b, s, {"floor": "white", "ceiling": "white",
                "back": "glossyback" if glossy_back else "white", "left": "red",
                "right": "green"})
    lo, hi, y = 0.35 * s, 0.65 * s, s - 0.01
    b.add_quad((lo, y, lo), (hi, y, lo), (hi, y, hi), (lo, y, hi), "lamp",
               emission=(17.0, 13.0, 6.0))
    return b.build()


def occluded_box(width: int = 8, height: int = 8) -> Scene:
    """Closed box whose camera chamber cannot see the lamp (src/scene.py:237-265)."""
    s = 4.0
    b = SceneBuilder()
    b.camera = Camera(_vec((s / 2, s / 2, 0.5)), _vec((s / 2, s / 2, s)), _vec((0, 1, 0)), 1.0,
                      width, height)
    b.add_material(Material("grey", _vec((0.5, 0.5, 0.5))))
    b.add_material(Material("lamp", np.zeros(3)))
    b.add_quad((0, 0, 0), (0, 0, s), (s, 0, s), (s, 0, 0), "grey")
    b.add_quad((0, s, 0), (s, s, 0), (s, s, s), (0, s, s), "grey")
    b.add_quad((0, 0, s), (0, s, s), (s, s, s), (s, 0, s), "grey")
    b.add_quad((0, 0, 0), (s, 0, 0), (s, s, 0), (0, s, 0), "grey")
    b.add_quad((0, 0, 0), (0, s, 0), (0, s, s), (0, 0, s), "grey")
    b.add_quad((s, 0, 0), (s, 0, s), (s, s, s), (s, s, 0), "grey")
    zd = s / 2 + 1.2
    b.add_quad((0, 0, zd), (0, s, zd), (s, s, zd), (s, 0, zd), "grey")
    y = s - 0.01
    b.add_quad((1, y, zd + 0.5), (3, y, zd + 0.5), (3, y, zd + 1.5), (1, y, zd + 1.5), "lamp",
               emission=(10.0, 10.0, 10.0))
    return b.build()


def corridor(width: int = 32, height: int = 32, length: float = 80.0, frames: int = 200,
             pan_speed: float = 0.35) -> Scene:
    """Floor/wall strip with a camera-attached lamp panning along +x (src/scene.py:268-290)."""
    b = SceneBuilder()
    b.camera = Camera(_vec((2.0, 1.5, -3.5)), _vec((2.0, 1.0, 0.0)), _vec((0, 1, 0)), 1.1,
                      width, height)
    b.add_material(Material("floor", _vec((0.6, 0.6, 0.55))))
    b.add_material(Material("wall", _vec((0.55, 0.5, 0.45))))
    b.add_material(Material("lamp", np.zeros(3)))
    b.add_quad((-5, 0, -6), (-5, 0, 3), (length, 0, 3), (length, 0, -6), "floor")
    b.add_quad((-5, 0, 3), (-5, 4, 3), (length, 4, 3), (length, 0, 3), "wall")
    b.add_quad((1.0, 3.2, -4.4), (3.0, 3.2, -4.4), (3.0, 3.2, -2.4), (1.0, 3.2, -2.4), "lamp",
               emission=(40.0, 40.0, 40.0))
    b.frames = frames
    v = _vec((pan_speed, 0.0, 0.0))
    b.motion = Motion(camera_velocity=v, light_velocity=v)
    return b.build()


def shadow_sweep(width: int = 40, height: int = 40, frames: int = 6,
                 light_velocity: float = 0.9) -> Scene:
    """Open room, a blocker and a strafing lamp (src/scene.py:293-320)."""
    s = 5.5
    b = SceneBuilder()
    b.camera = Camera(_vec((s / 2, 4.6, -7.0)), _vec((s / 2, 0.8, s / 2)), _vec((0, 1, 0)), 0.72,
                      width, height)
    b.add_material(Material("white", _vec((0.73, 0.73, 0.73))))
    b.add_material(Material("block", _vec((0.25, 0.25, 0.3))))
    b.add_material(Material("lamp", np.zeros(3)))
    _box(b, s, {"floor": "white", "back": "white"})
    x0, x1, z, h = 2.2, 3.3, 2.6, 2.2
    b.add_quad((x0, 0, z), (x0, h, z), (x1, h, z), (x1, 0, z), "block")
    b.add_quad((x0, 0, z + 0.15), (x1, 0, z + 0.15), (x1, h, z + 0.15), (x0, h, z + 0.15),
               "block")
    b.add_quad((0.4, 4.9, 2.0), (1.2, 4.9, 2.0), (1.2, 4.9, 2.8), (0.4, 4.9, 2.8), "lamp",
               emission=(90.0, 90.0, 90.0))
    b.frames = frames
    b.motion = Motion(light_velocity=_vec((light_velocity, 0.0, 0.0)))
    return b.build()


# The benchmark's closed box: camera inside, every primary ray hits a wall.
CLOSED_BOX = """\
camera 2.75 2.75 0.6  2.75 2.75 5.5  0 1 0  1.2 {width} {height}
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


def closed_box(width: int = 1920, height: int = 1080) -> Scene:
    return parse_scene(CLOSED_BOX.format(width=width, height=height))


_BUILTINS = {
    "cornell": cornell_box,
    "cornell-glossy": lambda **kw: cornell_box(glossy_back=True, **kw),
    "occluded": occluded_box,
    "corridor": corridor,
    "shadow-sweep": shadow_sweep,
    "closed-box": closed_box,
}


def load_scene(source: str, width: int | None = None, height: int | None = None) -> Scene:
    """A builtin scene by name, or a scene file (src/scene.py:333-347)."""
    kw = {k: v for k, v in (("width", width), ("height", height)) if v is not None}
    if source in _BUILTINS:
        return _BUILTINS[source](**kw)
    with open(source, "r", encoding="utf-8") as fh:
        scene = parse_scene(fh.read())
    if kw:
        scene.camera = replace(scene.camera, width=width or scene.camera.width,
                               height=height or scene.camera.height)
    return scene


def _numbers(tokens, n, what):
    if len(tokens) != n:
        raise SceneError(f"{what}: expected {n} numbers, got {len(tokens)}")
    try:
        return [float(x) for x in tokens]
    except ValueError as exc:
        raise SceneError(f"{what}: {exc}") from None


def _directive_camera(b, args):
    v = _numbers(args[:-2], 10, "camera")
    b.camera = Camera(_vec(v[0:3]), _vec(v[3:6]), _vec(v[6:9]), v[9], int(args[-2]),
                      int(args[-1]))


def _directive_material(b, args):
    rgb = _numbers(args[1:4], 3, "material albedo")
    extra = args[4:]
    gw = ge = 0.0
    if extra:
        if len(extra) != 3 or extra[0] != "glossy":
            raise SceneError("material: trailing tokens must be 'glossy W E'")
        gw, ge = float(extra[1]), float(extra[2])
    b.add_material(Material(args[0], _vec(rgb), gw, ge))


def _directive_polygon(b, args, corners):
    kind = "tri" if corners == 3 else "quad"
    pts = _numbers(args[:3 * corners], 3 * corners, kind)
    extra = args[3 * corners:]
    if not extra:
        raise SceneError(f"{kind}: missing material name")
    emission = (0.0, 0.0, 0.0)
    if len(extra) > 1:
        if len(extra) != 5 or extra[1] != "emit":
            raise SceneError(f"{kind}: trailing tokens must be 'emit R G B'")
        emission = tuple(float(x) for x in extra[2:5])
    corners_xyz = [pts[3 * i:3 * i + 3] for i in range(corners)]
    add = b.add_triangle if corners == 3 else b.add_quad
    add(*corners_xyz, material=extra[0], emission=emission)


def _directive_move(b, args):
    v = _vec(_numbers(args[1:], 3, "move"))
    if args[0] == "camera":
        b.motion.camera_velocity = v
    elif args[0] == "lights":
        b.motion.light_velocity = v
    else:
        raise SceneError(f"move: unknown target {args[0]!r}")


_DIRECTIVES = {
    "camera": _directive_camera,
    "material": _directive_material,
    "tri": lambda b, a: _directive_polygon(b, a, 3),
    "quad": lambda b, a: _directive_polygon(b, a, 4),
    "background": lambda b, a: setattr(b, "background", _vec(_numbers(a, 3, "background"))),
    "frames": lambda b, a: setattr(b, "frames", int(a[0])),
    "move": _directive_move,
    "emission_scale": lambda b, a: setattr(b.motion, "emission_scale", float(a[0])),
}


def parse_scene(text: str) -> Scene:
    """The line-based scene format (src/scene.py:359-421): '#' comments, one directive
    per line."""
    b = SceneBuilder()
    for lineno, raw in enumerate(text.splitlines(), start=1):
        tokens = raw.split("#", 1)[0].split()
        if not tokens:
            continue
        try:
            handler = _DIRECTIVES.get(tokens[0])
            if handler is None:
                raise SceneError(f"unknown directive {tokens[0]!r}")
            handler(b, tokens[1:])
        except (IndexError, ValueError) as exc:
            raise SceneError(f"line {lineno}: {exc}") from None
    return b.build()
