"""Full-size parity digests: run the REFERENCE on every BASELINE.json configuration that
fits one frame and commit SHA-256 digests of its outputs (tests/golden/fullsize.json).

Run in the build container (where the reference imports), never on the GPU box:

    PF_REFERENCE=baseline/_ref python tests/golden/make_fullsize.py

Configurations (BASELINE.json `configs`):
  cornell256  configs[0]: builtin cornell_box(256, 256), 1 spp, seed 1, first hit
  hd1         configs[1]: closed box 1920x1080, 1 spp, first hit (select_k 1, rr_start 9)
  hd4         configs[2]: the same scene, select_k 1..4 concatenated with sample += k-1
              (8,184,972 vertices -- the benchmark's stream)
  hd1_filter  configs[3]: hd1's stream, 8 frames of temporal_mode "filter" with the
              animated-scene seed schedule mix64(1 ^ f*G) and begin_frame(f) each frame
              (src/pipeline.py:329-333)
  hd4_seq     the benchmark's frame sequence: configs[2]'s stream, 4 integrate-mode
              frames with the animated seed schedule bench.py uses (tables at frames 0, 3)
  hd1_filter64  configs[3] as named: the same for 64 frames (tables digested at frames
              0, 7, 15, 31, 47, 63; sources, means and image every frame)

Everything digested is produced by the reference's own code path (trace,
vertex_keys, accumulate_phase, resolve_phase, VoxelTable); this script only hashes it
(oracle/digest.py, shared with the GPU tests).
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
REF = os.environ.get("PF_REFERENCE", os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, os.path.abspath(REF))
sys.path.insert(0, ROOT)

import pathfilter as pf  # noqa: E402
from pathfilter import rng as prng  # noqa: E402
from pathfilter.keys import FilterConfig  # noqa: E402
from pathfilter.pipeline import FrameState, accumulate_phase, resolve_phase, vertex_keys  # noqa: E402
from pathfilter.scene import parse_scene  # noqa: E402
from pathfilter.tracer import TraceOptions, VertexStream, trace  # noqa: E402

from oracle.digest import composite, digest, table_digest  # noqa: E402

assert pf.BACKEND == "native", "build the reference's Cython extension first"

STREAM_FIELDS = ("position", "normal", "omega_r", "contribution", "throughput", "pixel",
                 "sample", "layer_id", "camera_distance")
KEY_FIELDS = ("qx", "qy", "qz", "level", "aux", "index", "fingerprint", "jittered")
THREADS = os.cpu_count() or 1

CLOSED_BOX = open(os.path.join(HERE, "make_golden.py")).read().split('CLOSED_BOX = """')[1] \
    .split('"""')[0]


def next_pow2(n: int) -> int:
    return 1 << (int(n) - 1).bit_length()


def stream_digests(vs) -> dict:
    return {f: digest(getattr(vs, f)) for f in STREAM_FIELDS}


def key_digests(k) -> dict:
    return {f: digest(getattr(k, f)) for f in KEY_FIELDS}


def box_stream(w, h, ks):
    scene = parse_scene(CLOSED_BOX.format(w=w, h=h))
    parts, base = [], None
    for k in ks:
        tr = trace(scene, spp=1, seed=1, options=TraceOptions(select_k=k, rr_start=9),
                   threads=THREADS)
        vs = tr.vertices
        vs.sample = vs.sample + (k - 1)
        parts.append(vs)
        if k == 1:
            base = tr.base_image
    return scene, VertexStream.concat(parts), base


def filter_frames(scene, vs, base, frames=1, mode="integrate", animated=False,
                  table_frames=None):
    """begin_frame + accumulate_phase + resolve_phase per frame (render_frame minus the
    tracer, src/pipeline.py:321-363) on a fresh FrameState.  table_frames: the frames
    whose tables are digested (default: all)."""
    h, w = base.shape[:2]
    cfg = FilterConfig(capacity=next_pow2(2 * w * h), temporal_mode=mode).for_camera(
        scene.camera.fov, scene.camera.height)
    state = FrameState.from_config(cfg)
    out = {"cfg": {k: getattr(cfg, k) for k in cfg.__dataclass_fields__}, "frames": []}
    for f in range(frames):
        seed = prng.mix64(1 ^ (f * 0x9E3779B97F4A7C15)) if animated else 1
        t0 = time.perf_counter()
        state.fine.begin_frame(f, cfg)
        state.coarse.begin_frame(f, cfg)
        fk, ck, stats = accumulate_phase(vs, cfg, state, f, seed)
        image, report = resolve_phase(vs, cfg, state, f, seed, 1, base, fk)
        dt = time.perf_counter() - t0
        rec = {"seed": str(seed), "seconds": round(dt, 2),
               "source": digest(report.source),
               "source_counts": np.bincount(report.source, minlength=4).tolist(),
               "chosen": digest(report.means), "image": digest(image),
               "probe_failures": int(stats.probe_failures),
               "coarse_probe_failures": int(stats.coarse_probe_failures)}
        if table_frames is None or f in table_frames:
            for name, t in (("fine", state.fine), ("coarse", state.coarse)):
                rec[name] = table_digest({k: getattr(t, k) for k in
                                          ("tags", "sums", "counts", "hist_sums", "hist_counts",
                                           "last_touch", "deltas")})
        # the composite restated over the reference's own chosen means reproduces its image
        assert digest(composite(base, vs.pixel, vs.throughput, report.means, 1)) == rec["image"]
        if f == 0:
            rec["keys"] = {"fine": key_digests(fk), "coarse": key_digests(ck),
                           "lookup": key_digests(vertex_keys(vs, cfg, seed,
                                                             prng.STREAM_JITTER_LOOKUP))}
        out["frames"].append(rec)
        print(f"  frame {f}: {dt:.1f} s, sources {rec['source_counts']}", flush=True)
    return out


def main():
    res = {"meta": {"generator": "tests/golden/make_fullsize.py",
                    "reference": "pathfilter " + pf.__version__, "backend": pf.BACKEND,
                    "numpy": np.__version__, "python": platform.python_version(),
                    "libc": " ".join(platform.libc_ver()), "threads": THREADS}}
    only = set(sys.argv[1:])

    def want(name):
        return not only or name in only

    if want("cornell256"):
        print("cornell256", flush=True)
        scene = pf.cornell_box(256, 256)
        tr = trace(scene, spp=1, seed=1, options=TraceOptions(select_k=1), threads=THREADS)
        vs, base = tr.vertices, tr.base_image
        res["cornell256"] = {"n": len(vs), "stream": stream_digests(vs), "base": digest(base),
                             **filter_frames(scene, vs, base)}
    if want("hd1") or want("hd1_filter"):
        print("hd1", flush=True)
        scene, vs, base = box_stream(1920, 1080, [1])
        if want("hd1"):
            res["hd1"] = {"n": len(vs), "stream": stream_digests(vs), "base": digest(base),
                          **filter_frames(scene, vs, base)}
        if want("hd1_filter"):
            print("hd1_filter", flush=True)
            res["hd1_filter"] = {"n": len(vs), "stream": stream_digests(vs),
                                 **filter_frames(scene, vs, base, frames=8, mode="filter",
                                                 animated=True)}
    if want("hd1_filter64"):
        print("hd1_filter64", flush=True)
        scene, vs, base = box_stream(1920, 1080, [1])
        res["hd1_filter64"] = {"n": len(vs), "stream": stream_digests(vs),
                               **filter_frames(scene, vs, base, frames=64, mode="filter",
                                               animated=True,
                                               table_frames={0, 7, 15, 31, 47, 63})}
    if want("hd4_seq"):
        print("hd4_seq", flush=True)
        scene, vs, base = box_stream(1920, 1080, [1, 2, 3, 4])
        res["hd4_seq"] = {"n": len(vs), "stream": stream_digests(vs), "base": digest(base),
                          **filter_frames(scene, vs, base, frames=4, animated=True,
                                          table_frames={0, 3})}
    if want("hd4"):
        print("hd4", flush=True)
        scene, vs, base = box_stream(1920, 1080, [1, 2, 3, 4])
        res["hd4"] = {"n": len(vs), "stream": stream_digests(vs), "base": digest(base),
                      **filter_frames(scene, vs, base)}
    path = os.path.join(HERE, "fullsize.json")
    old = json.load(open(path)) if os.path.exists(path) and only else {}
    old.update(res)
    with open(path, "w") as f:
        json.dump(old, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
