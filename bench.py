"""Benchmark: filtered path vertices/s (insert + query) for one HD 1 spp 4-bounce frame.

Workload (BASELINE.json configs[2]): 1920x1080, 1 spp, all
vertices of 4-bounce paths in the closed Cornell box of SURVEY App. B, traced on the
device by the repo's path tracer exactly as the reference's recipe does (select_k =
1..4, rr_start 9, seed 1, sample += k-1: 8,184,972 vertices, bit-identical to the
reference tracer's stream); `--stream synthetic` uses streams.closed_box_stream
instead.  Capacity next_pow2(2*W*H) = 2^22, fine + coarse tables,
FilterConfig defaults (jitter, fixed-point sums, integrate).  One step = one frame:
begin_frame on both tables, accumulate_phase (keys + insert), resolve_phase
(ladder + composite), with the animated-scene seed schedule (src/pipeline.py:329).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line (rank 0).  N>1 (torchrun, NCCL) runs the key-sharded frame
(paper_1902_05942_b200/sharded.py): rank r traces its own sample of every
pixel (1 spp per GPU, spp = N for the image), the global fine/coarse tables of
capacity 2^22 are split into N owner slices, pre-aggregated records move by
all-to-all, the owners' cells by all-gather into a per-rank replica, and the flat
image by reduce-scatter.  Weak scaling: 8.18 M vertices per GPU per frame.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_PIX, H_PIX, BOUNCES = 1920, 1080, 4
TEMPORAL = "integrate"
# --workload: the default is the metric's configuration (BASELINE.json configs[2]); the
# others are the remaining configs of BASELINE.json, for the record
WORKLOADS = {
    "hd4": (1920, 1080, 4, "integrate", "configs[2]"),
    "hd1": (1920, 1080, 1, "integrate", "configs[1]"),
    "hd-temporal": (1920, 1080, 1, "filter", "configs[3]: EMA blend + aging, one step = one frame"),
    "uhd4": (3840, 2160, 4, "integrate", "configs[4] on one GPU"),
    # configs[4] as named: ONE 4K frame split into N pixel-row bands (rank r traces rows
    # [r H/N, (r+1) H/N)), key-sharded C = 2^24 tables, band composite: strong scaling
    "uhd4-band": (3840, 2160, 4, "integrate", "configs[4]: 4K frame in N row bands"),
}
METRIC = "filtered path vertices/sec (insert+query); ms/frame at 1080p 1spp 4 bounces"
WORKLOAD = "1920x1080 1spp, all vertices of 4-bounce paths (closed Cornell box, synthetic)"


def make_stream(kind: str, rank: int = 0, device=None, world: int = 1, band: bool = False):
    """(stream dict of CUDA tensors, base image) of the benchmark workload for a rank:
    rank r traces sample r of every pixel (distinct path ids and jitter draws); with
    `band`, rank r traces sample 0 of its pixel-row band and the base image is the band."""
    from paper_1902_05942_b200.streams import closed_box_stream
    if band and world > 1:
        from paper_1902_05942_b200.scene import closed_box
        from paper_1902_05942_b200.tracer import band_stream
        if H_PIX % world:
            raise SystemExit(f"--workload uhd4-band needs H={H_PIX} divisible by --gpus")
        rows = H_PIX // world
        vs, base = band_stream(closed_box(W_PIX, H_PIX), BOUNCES, 1, rank * rows,
                               (rank + 1) * rows)
        return {f: getattr(vs, f).contiguous() for f in FIELDS}, base.contiguous()
    if kind == "synthetic":
        stream, base = closed_box_stream(W_PIX, H_PIX, BOUNCES, 1 + rank, device=device)
        if rank:
            stream["sample"] = stream["sample"] + rank * BOUNCES
            base = closed_box_stream(W_PIX, H_PIX, 1, 1, device=device)[1]
        return stream, base
    from paper_1902_05942_b200.scene import closed_box
    from paper_1902_05942_b200.tracer import multi_bounce_stream
    vs, base = multi_bounce_stream(closed_box(W_PIX, H_PIX), BOUNCES, 1,
                                   sample_offset=BOUNCES * rank)
    if rank:  # the image's base term: the k = 1 trace of sample 0, identical on every rank
        base = multi_bounce_stream(closed_box(W_PIX, H_PIX), 1, 1)[1]
    stream = {f: getattr(vs, f).contiguous() for f in FIELDS}
    return stream, base.contiguous()
# algorithmic HBM bytes
INSERT_BYTES_PER_VERTEX = 96      # position 24 + normal 24 + distance 8 + pixel 8 + sample 8 + contribution 24
QUERY_BYTES_PER_VERTEX = 120      # + throughput 24
QUERY_BYTES_PER_PIXEL = 48        # base image read 24 + filtered image write 24
MARK_EVERY = 5                    # timed frames with phase events: 0, 5, 10, ...

_REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                0x100: "display_clock_setting"}


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._proc = None
        self._thread = None

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._thread = threading.Thread(target=self._read, daemon=True)
            self._thread.start()
        except OSError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16),
                                         time.time()))
                except ValueError:
                    pass

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self._proc is not None and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.02)

    def window(self, t0, t1):
        """Keep the samples taken inside [t0, t1] (plus the nearest one if none)."""
        inside = [s for s in self.samples if t0 <= s[3] <= t1]
        if not inside and self.samples:
            inside = [min(self.samples, key=lambda s: abs(s[3] - (t0 + t1) / 2))]
        self.samples = inside

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(s[0] for s in self.samples)
        reasons = 0
        for s in self.samples:
            reasons |= s[2]
        names = [v for k, v in _REASON_BITS.items() if reasons & k and v != "gpu_idle"]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": names, "samples": len(self.samples)}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _traffic(kernel: str, workload: str, stream: str = "traced"):
    """dram bytes (or, for "<kernel>_inst", warp instructions) per launch from the
    committed ncu --set full capture OF THIS WORKLOAD (profiles/ncu_traffic.json is keyed
    by bench workload), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if stream != "traced" or not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh).get(workload, {}).get(kernel)


def _l2_red_peak():
    """Sustained random-address RED.U64 rate (ops/s) measured by tools/l2atomics.cu."""
    p = os.path.join(ROOT, "profiles", "r1_l2atomics.log")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        for line in fh:
            d = json.loads(line)
            if d.get("pattern") == "red_u64_random":
                return d["gops_per_s"] * 1e9
    return None


def make_config(pf):
    from paper_1902_05942_b200.streams import camera_footprint
    cap = 1 << (2 * W_PIX * H_PIX - 1).bit_length()
    return pf.FilterConfig(capacity=cap, footprint_scale=camera_footprint(H_PIX),
                           temporal_mode=TEMPORAL)


def workload_text(kind: str) -> str:
    if kind == "synthetic":
        return WORKLOAD
    return (f"{W_PIX}x{H_PIX} 1spp, all vertices of {BOUNCES}-bounce paths: SURVEY App. B closed "
            f"box traced on device (select_k 1..{BOUNCES}, rr_start 9, seed 1), "
            f"temporal_mode {TEMPORAL}")


# The benchmark scene, as scene text for the reference's own parser.  The
# reference arm must not import this repo's package (it loads libpf_b200.so), so the
# text is restated here; tests/test_bench_cpu.py checks it equals scene.CLOSED_BOX.
REF_CLOSED_BOX = """\
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
GOLDEN = 0x9E3779B97F4A7C15


def reference_module():
    """The unmodified reference installed in baseline/_ref (native Cython backend), or
    None.  Imported from its install directory only -- never this repo's package."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "pathfilter")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import pathfilter
        import pathfilter.pipeline  # noqa: F401
        return pathfilter
    except Exception as exc:  # noqa: BLE001
        print(f"bench: reference import failed ({exc})", file=sys.stderr)
        return None


def reference_config(ref, scene, temporal):
    """The reference's FilterConfig for a camera: defaults, capacity next_pow2(2 W H)
    (src/cli.py:142-143), footprint from the camera (src/keys.py:74-76)."""
    cam = scene.camera
    cap = 1 << (2 * cam.width * cam.height - 1).bit_length()
    return ref.FilterConfig(capacity=cap, temporal_mode=temporal).for_camera(cam.fov, cam.height)


def reference_stream(ref, width, height, bounces, threads):
    """The benchmark stream traced by the REFERENCE's tracer (src/tracer.py:411-461):
    select_k = 1..bounces at 1 spp, seed 1, rr_start 9, sample += k - 1, concatenated
    (SURVEY App. B).  Returns (scene, VertexStream, base image of k = 1)."""
    from pathfilter.scene import parse_scene
    from pathfilter.tracer import TraceOptions, VertexStream, trace
    scene = parse_scene(REF_CLOSED_BOX.format(width=width, height=height))
    parts, base = [], None
    for k in range(1, bounces + 1):
        tr = trace(scene, spp=1, seed=1, options=TraceOptions(select_k=k, rr_start=9),
                   threads=threads)
        v = tr.vertices
        v.sample = v.sample + (k - 1)
        parts.append(v)
        if base is None:
            base = tr.base_image
    return scene, VertexStream.concat(parts), base


def reference_frame(ref, vs, base, cfg, state, frame, threads):
    """One frame of the reference's own CPU path: begin_frame on both tables,
    accumulate_phase, resolve_phase (src/pipeline.py:321-363 minus the tracer), with the
    animated-scene seed schedule (src/pipeline.py:329).  Returns seconds."""
    seed = ref.rng.mix64(1 ^ ((frame * GOLDEN) & 0xFFFFFFFFFFFFFFFF))
    t0 = time.perf_counter()
    state.fine.begin_frame(frame, cfg)
    state.coarse.begin_frame(frame, cfg)
    fk, _, _ = ref.pipeline.accumulate_phase(vs, cfg, state, frame, seed, threads=threads)
    ref.pipeline.resolve_phase(vs, cfg, state, frame, seed, 1, base, fk)
    return time.perf_counter() - t0


class _Sub:
    def __len__(self):
        return len(self.pixel)


FIELDS = ("position", "normal", "omega_r", "contribution", "throughput", "pixel", "sample",
          "layer_id", "camera_distance")


def host_sample(stream_np, stride: int):
    s = _Sub()
    for f in FIELDS:
        setattr(s, f, np.ascontiguousarray(getattr(stream_np, f)[::stride]))
    return s


def port_baseline(stream_np, base_np, cfg_kwargs, frames: int, stride: int):
    """Fallback when baseline/_ref is absent: the oracle port (oracle/pf_oracle.py, one
    thread) on every `stride`-th vertex."""
    from oracle import pf_oracle
    cfg = pf_oracle.Config(**{k: v for k, v in cfg_kwargs.items()
                              if k in pf_oracle.Config.__dataclass_fields__})
    state = pf_oracle.State.from_config(cfg)
    sample = host_sample(stream_np, stride)
    times = []
    for f in range(frames):
        seed = pf_oracle.mix64(1 ^ ((f * GOLDEN) & 0xFFFFFFFFFFFFFFFF))
        t0 = time.perf_counter()
        pf_oracle.filter_frame(sample, cfg, state, f, seed, 1, base_np)
        times.append(time.perf_counter() - t0)
    return len(sample.pixel), times


def cpu_baseline_leg(stream_np, base_np, cfg, frames: int = 2):
    """cpu_baseline of the b200 arm: the unmodified reference (native backend, every host
    thread) filtering the FULL frame of the same stream (the device tracer's stream,
    bit-identical to the reference tracer's -- tests/test_gpu_fullsize.py); the best of
    `frames` consecutive frames.  Falls back to the oracle port on a stride sample."""
    ref = reference_module()
    threads = os.cpu_count() or 1
    if ref is None:
        kwargs = dict(capacity=cfg.capacity, footprint_scale=cfg.footprint_scale,
                      temporal_mode=cfg.temporal_mode)
        n, times = port_baseline(stream_np, base_np, kwargs, frames, 4)
        return {"value": n / min(times), "unit": "vertices/s", "cores": 1, "kind": "port",
                "sample": f"every 4th vertex of the same stream ({n} vertices), oracle port, "
                          f"best of {frames} frames"}
    vs = ref.VertexStream(**{f: np.ascontiguousarray(getattr(stream_np, f)) for f in FIELDS})
    rcfg = ref.FilterConfig(capacity=cfg.capacity, footprint_scale=cfg.footprint_scale,
                            temporal_mode=cfg.temporal_mode)
    state = ref.FrameState.from_config(rcfg)
    times = [reference_frame(ref, vs, base_np, rcfg, state, f, threads) for f in range(frames)]
    n = len(vs)
    return {"value": n / min(times), "unit": "vertices/s", "cores": threads,
            "kind": "reference",
            "sample": f"the full frame ({n} vertices, C={cfg.capacity} fine+coarse), best of "
                      f"{frames} consecutive frames, baseline/_ref backend={ref.BACKEND}, "
                      f"threads={threads} (numpy key build single-threaded)",
            "frame_s": times}


def run_reference_arm(args):
    """The reference arm: the UNMODIFIED reference (baseline/_ref) on the same workload --
    its own tracer builds the input, its own accumulate_phase + resolve_phase filter the
    full frame every step.  This process never imports this repo's package."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    ref = reference_module()
    threads = os.cpu_count() or 1
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "baseline/_ref (the reference's install) is missing or does not "
                          "import"}), flush=True)
        return 0
    t0 = time.perf_counter()
    scene, vs, base = reference_stream(ref, W_PIX, H_PIX, BOUNCES, threads)
    trace_s = time.perf_counter() - t0
    cfg = reference_config(ref, scene, TEMPORAL)
    state = ref.FrameState.from_config(cfg)
    n = len(vs)
    # the CPU frame takes seconds: at most two untimed warm-up frames
    warm = min(args.warmup, 2)
    for f in range(warm):
        reference_frame(ref, vs, base, cfg, state, f, threads)
    times = [reference_frame(ref, vs, base, cfg, state, warm + k, threads)
             for k in range(args.steps)]
    per = sum(times) / len(times)
    value = n / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "vertices/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_text("traced").replace("traced on device",
                                                               "traced by the reference"),
                   "bench_workload": args.workload,
                   "vertices_per_frame": n, "pixels": W_PIX * H_PIX,
                   "capacity": cfg.capacity, "tables": "fine+coarse",
                   "temporal_mode": cfg.temporal_mode, "sum_mode": cfg.sum_mode,
                   "input": f"traced by the reference's own tracer ({threads} threads, "
                            f"{trace_s:.1f} s, untimed)",
                   "warmup_run": warm},
        "cpu_baseline": {"value": value, "unit": "vertices/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"the full frame every step ({n} vertices), backend="
                                   f"{ref.BACKEND}, threads={threads} (numpy key build "
                                   f"single-threaded)"},
        "e2e": {"value": value, "unit": "vertices/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "frame_s": times,
        "native_so": sorted({os.path.basename(p) for p in _loaded_libs()}),
    }
    print(json.dumps(line), flush=True)
    return 0


def _loaded_libs():
    """Shared objects this process has mapped that belong to this repo or the reference
    install (a provenance record: the reference arm must map none of the repo's)."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                p = line.split()[-1] if line.strip() else ""
                if p.endswith(".so") and p.startswith(ROOT):
                    out.add(p)
    except OSError:
        pass
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if world > 1:
        # NCCL's init lines (rank count per communicator) in the log, however the ranks
        # were launched
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # PF_BENCH_BACKEND=gloo + PF_BENCH_ONE_DEVICE=1: exercise the N-rank code path on a
        # single GPU (exchanges through host memory, no kernel waits on another rank);
        # numbers from such a run are not multi-GPU measurements
        dist.init_process_group(os.environ.get("PF_BENCH_BACKEND", "nccl"))
    if os.environ.get("PF_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)

    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    import paper_1902_05942_b200 as pf
    from paper_1902_05942_b200 import _lib, rng
    from paper_1902_05942_b200.streams import stream_to_numpy

    cfg = make_config(pf)
    band = args.workload == "uhd4-band"
    stream, base = make_stream(args.stream, rank, world=world, band=band)
    vs = pf.VertexStream(**stream)
    n = len(vs)
    n_pix = int(base.shape[0]) * int(base.shape[1])   # this rank's pixels
    composite, pixel_base = ("band", rank * n_pix) if band else ("reduce", 0)
    n_total = n * world
    if world > 1:  # vertices of the whole job (band ranks differ)
        t = torch.tensor([n], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        n_total = int(t.item())
    if world > 1:
        from paper_1902_05942_b200 import sharded
        state = sharded.ShardedState(cfg, rank, world, agg_capacity=1 << 20)
    else:
        state = pf.FrameState.from_config(cfg)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    phases = ({"begin_check": [], "insert": [], "resolve": []} if world == 1 else
              {"begin_keys": [], "exchange_apply_publish": [], "resolve_image": []})

    def step(f, evs=None):
        # one frame = ONE pf_filter_frame call; its phase events (recorded inside the C
        # call on the launching stream) bracket begin+check, the insert kernel, resolve
        seed = rng.frame_seed(1, f)
        if world > 1:
            sharded.run_dist(sharded.filter_frame_sharded(
                vs, base, cfg, state, 1 if band else world, seed, pixel_base=pixel_base,
                composite=composite, want_means=True,
                phase_events=evs))
        else:
            pf.filter_frame(vs, base, cfg, state, 1, seed, want_means=True, phase_events=evs)

    clocks = ClockSampler(local)
    clocks.__enter__()
    clocks.wait_first()
    for f in range(args.warmup):
        step(f)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # phase events on every MARK_EVERY-th timed frame (4 event records cost a frame
    # ~17 us: they break the kernels' programmatic-launch overlap), created and
    # materialised (one record each) before the timed region, so inside it only the C
    # call's own records remain
    marked = [k for k in range(args.steps) if k % MARK_EVERY == 0]
    marks = {k: tuple(ev() for _ in range(4)) for k in marked}
    for m in marks.values():
        for e in m:
            e.record()
    torch.cuda.synchronize()
    start, stop = ev(), ev()
    t_wall0 = time.time()
    start.record()
    for k in range(args.steps):
        step(args.warmup + k, marks.get(k))
    stop.record()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    time.sleep(0.05)
    clocks.__exit__(None, None, None)
    clocks.window(t_wall0 - 0.05, t_wall1 + 0.05)
    if world > 1:
        dist.barrier()
    elapsed = start.elapsed_time(stop) / 1e3
    t_max = elapsed
    if world > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    names = list(phases)
    for e0, e1, e2, e3 in marks.values():
        phases[names[0]].append(e0.elapsed_time(e1))
        phases[names[1]].append(e1.elapsed_time(e2))
        phases[names[2]].append(e2.elapsed_time(e3))
    ph = {k: float(np.mean(v)) for k, v in phases.items()}
    value = n_total * args.steps / t_max
    ms_per_step = t_max / args.steps * 1e3

    # roofline of the dominant phase kernel (bytes per launch / mean launch time)
    peak, peak_kind = _peaks()
    if world > 1:  # the round-1 key + pre-aggregation kernel reads the insert inputs
        kname, kbytes = "shard_keys_kernel", INSERT_BYTES_PER_VERTEX * n
        kms = ph["begin_keys"]
    elif ph["insert"] >= ph["resolve"]:
        kname, kbytes, kms = "insert_frame_kernel", INSERT_BYTES_PER_VERTEX * n, ph["insert"]
    else:
        kname, kbytes, kms = ("resolve_phase", QUERY_BYTES_PER_VERTEX * n +
                              QUERY_BYTES_PER_PIXEL * n_pix, ph["resolve"])
    achieved = kbytes / (kms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "bytes_per_launch": kbytes, "traffic": _traffic(kname, args.workload, args.stream)}

    # the insert kernel is issue-bound, not HBM-bound: its instruction issue rate against
    # the SMs' peak (148 SMs x 4 schedulers x 1 warp-instruction per clock), with the
    # per-launch instruction count from the committed ncu capture (same workload)
    issue = None
    inst = (_traffic("insert_frame_kernel_inst", args.workload, args.stream)
            if kname == "insert_frame_kernel" else None)
    if inst:
        sm_mhz = clocks.summary().get("sm_mhz") or 1965.0
        ipeak = 148 * 4 * sm_mhz * 1e6
        iach = inst / (kms / 1e3)
        issue = {"bound": "issue", "kernel": kname, "achieved": iach, "peak": ipeak,
                 "unit": "warp-inst/s", "frac": iach / ipeak, "inst_per_launch": inst}
    # and its L2 reductions against the sustained random-address RED rate measured by
    # tools/l2atomics.cu on this pool (profiles/r1_l2atomics.log)
    atomics = None
    reds = (_traffic("insert_frame_kernel_red_sectors", args.workload, args.stream)
            if kname == "insert_frame_kernel" else None)
    red_peak = _l2_red_peak()
    if reds and red_peak:
        rach = reds / (kms / 1e3)
        atomics = {"bound": "l2_atomics", "kernel": kname, "achieved": rach, "peak": red_peak,
                   "unit": "red/s", "frac": rach / red_peak, "red_per_launch": reds}

    # per-rank bytes of a frame (world > 1): the algorithmic HBM bytes of this rank's
    # vertices and pixels, and what crossed the interconnect in the last timed frame
    comm = None
    if world > 1 and getattr(state, "last_comm", None) is not None:
        c = {k: int(v) for k, v in state.last_comm.items()}
        t = torch.tensor([sum(c.values())], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        comm = {"rank0_bytes_per_frame": c, "rank0_total": sum(c.values()),
                "max_rank_total": int(t.item()),
                "hbm_algorithmic_bytes_per_rank": INSERT_BYTES_PER_VERTEX * n +
                QUERY_BYTES_PER_VERTEX * n + QUERY_BYTES_PER_PIXEL * n_pix}

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(pf, rng, cfg, stream, base, args, n, rank, world, composite, pixel_base,
                      n_total)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_leg(stream_to_numpy(stream), base.cpu().numpy(), cfg)

    in_bytes = QUERY_BYTES_PER_VERTEX * n + QUERY_BYTES_PER_PIXEL * n_pix
    if rank == 0:
        # single: prologue, insert, effective records (+ image = base / work-counter
        # init), resolve main, fallback keys, pool (spp = 1: the composite lands in the
        # image, no finalize).  sharded: begin x2, check, keys, emit, apply, reset,
        # publish x2, replica clear + write, resolve main, fallback keys, pool, finalize
        # (NCCL kernels not counted)
        launches = (6 if world == 1 else 15) * args.steps
        line = {
            "metric": METRIC, "value": value, "unit": "vertices/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if band else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_text(args.stream), "bench_workload": args.workload,
                       "vertices_per_frame": n_total, "vertices_rank0": n,
                       "pixels": n_pix * (world if band else 1),
                       "capacity": cfg.capacity, "tables": "fine+coarse",
                       "temporal_mode": cfg.temporal_mode, "sum_mode": cfg.sum_mode,
                       "parallelism": (f"key-sharded tables x{world} (NCCL all-to-all), "
                                       f"1 spp per GPU" if world > 1 else "single"),
                       "l2": f"inputs {in_bytes / 1e9:.2f} GB per frame > 126 MB L2 "
                             "(no flush needed)",
                       "outputs": "filtered image + per-vertex source and chosen mean "
                                  "(the reference's ResolveReport)",
                       # where the implementation departs from the north-star sketch, each
                       # measured
                       "design": {
                           "fused_insert_warp_merge": "off: __match_any_sync merging of equal "
                                                      "keys measured slower (insert 0.93 vs "
                                                      "0.82 ms); kept in the batch and shard "
                                                      "inserts",
                           "vertex_loads": "per-lane 8-byte loads with an L2 evict_first "
                                           "policy; a TMA (cp.async.bulk) tile pipeline "
                                           "measured slower (1.22 vs 1.06 ms)",
                           "table_layout": "dense tags and counts, channel-major live sums, "
                                           "64-byte cold records; 32 MB L2 set-aside for "
                                           "evict_last table / composite lines",
                           "kernel_chain": "6 kernels per frame with programmatic dependent "
                                           "launch"}},
            "phases_ms": ph, "roofline": roofline, "roofline_issue": issue, "comm": comm,
            "roofline_atomics": atomics, "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks.summary(),
            "build": {"library": os.path.relpath(_lib.LIB_PATH, ROOT), "build_id": _lib.build_id(),
                      "tree_id": _lib.source_id()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(pf, rng, cfg, stream, base, args, n, rank=0, world=1, composite="reduce",
            pixel_base=0, n_total=None):
    """Same frame through the public API from pinned host buffers: H2D of every
    input the frame reads, the frame, D2H of the filtered image (this rank's rows for
    N > 1) -- all timed; max over ranks.  One GPU: pf.HostFramePipeline, whose copy
    stream moves frame f+1's inputs while frame f computes (each step still carries its
    own H2D and D2H inside the timed region)."""
    import torch
    import torch.distributed as dist
    fields = ("position", "normal", "contribution", "throughput", "pixel", "sample",
              "camera_distance")
    host = {f: stream[f].cpu().pin_memory() for f in fields}
    hbase = base.cpu().pin_memory()
    himg = torch.empty_like(hbase).pin_memory()
    if world > 1:
        dev = {f: torch.empty_like(stream[f]) for f in fields}
        dbase = torch.empty_like(base)
        unused = {"omega_r": torch.zeros_like(stream["position"]),
                  "layer_id": torch.zeros_like(stream["pixel"])}
        from paper_1902_05942_b200 import sharded
        state = sharded.ShardedState(cfg, rank, world, agg_capacity=1 << 20)
        if composite == "reduce":
            himg = himg[: himg.shape[0] // world]
    else:
        state = pf.FrameState.from_config(cfg)
    h2d = sum(t.numel() * t.element_size() for t in host.values()) + hbase.numel() * 8
    d2h = himg.numel() * 8

    from types import SimpleNamespace
    hvs = SimpleNamespace(**host)
    pipe = pf.HostFramePipeline(cfg, state) if world == 1 else None

    def frame(f, start=None):
        if pipe is not None:  # single GPU: the public host-buffer API, copies overlapped
            pipe.submit(hvs, hbase, 1, rng.frame_seed(1, f), start_event=start)
            return
        for k in fields:
            dev[k].copy_(host[k], non_blocking=True)
        dbase.copy_(hbase, non_blocking=True)
        vs = pf.VertexStream(**dev, **unused)
        image, _, _ = sharded.run_dist(sharded.filter_frame_sharded(
            vs, dbase, cfg, state, 1 if composite == "band" else world, rng.frame_seed(1, f),
            pixel_base=pixel_base, composite=composite))
        himg.copy_(image, non_blocking=True)

    for f in range(max(1, min(args.warmup, 3))):
        frame(f)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(1, min(args.steps, 10))
    s.record()
    for f in range(k):
        frame(100 + f, s if f == 0 else None)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    if world > 1:
        tt = torch.tensor([t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    # the bound: the host-to-device direction (the read-back overlaps it on the other
    # copy engine) -- the step's H2D bytes as one pinned copy, best of 3, no frame
    big_h = torch.empty(h2d // 8, dtype=torch.float64).pin_memory()
    big_d = torch.empty(h2d // 8, dtype=torch.float64, device="cuda")
    copy_t = []
    for _ in range(3):
        s.record()
        big_d.copy_(big_h, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        copy_t.append(s.elapsed_time(e) / 1e3)
    del big_h, big_d
    per = t / k
    return {"value": (n_total or n * world) * k / t, "unit": "vertices/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": per * 1e3, "steps": k,
            "roofline": {"bound": "pcie_h2d", "achieved": h2d / per / 1e9,
                         "peak": h2d / min(copy_t) / 1e9, "unit": "GB/s",
                         "peak_kind": "measured on this box: the step's H2D bytes as one "
                                      "pinned copy",
                         "frac": min(copy_t) / per}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--workload", default="hd4", choices=list(WORKLOADS),
                    help="BASELINE.json configuration (default: the metric's, configs[2])")
    ap.add_argument("--stream", default="traced", choices=["traced", "synthetic"],
                    help="benchmark input: App. B scene traced on device, or the synthetic "
                         "closed-box generator")
    ap.add_argument("--dry-run", action="store_true",
                    help="start the ranks, one barrier + all-reduce, print the rank count "
                         "(tests the launch path; no GPU work)")
    args = ap.parse_args()
    global W_PIX, H_PIX, BOUNCES, TEMPORAL
    W_PIX, H_PIX, BOUNCES, TEMPORAL, _ = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference_arm(args)
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if int(world or 1) != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to "
                         "report a rank count other than the one asked for")
    if args.dry_run:
        return dry_run(args)
    return run_b200(args)


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-execute this command under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous, a free port),
    NCCL_DEBUG=INFO (init lines only) so the rank count is visible in the log."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def dry_run(args) -> int:
    import torch
    import torch.distributed as dist
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    n = world
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        t = torch.ones(1)
        if torch.cuda.is_available():
            torch.cuda.set_device(_env_int("LOCAL_RANK", 0))
            t = t.cuda()
        dist.all_reduce(t)
        n = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_reduced": n}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
