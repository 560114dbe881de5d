"""SPEC acceptance criteria measured on the device path (the reference states them for
its CPU implementation, SPEC.md "ACCEPTANCE CRITERIA").

- Criterion 3 (variance reduction, the paper's Fig. 1 analogue) and the jitter half of
  criterion 8: Cornell box, 1 spp filtered vs 1 spp unfiltered against a 1024-spp image
  of the same tracer, pixel-centred rays (the reference's image-error fixture,
  pkg/tests/conftest.py:17-26).  Filtered MSE >= 3x lower; jitter on costs <= 1.5x the
  jitter-off MSE.
- Criterion 6 (constant-time scaling, paper 3.3.1) in the reference's bench mode
  (src/bench.py via paper_1902_05942_b200.bench): per-vertex time of accumulate_batch +
  lookup_slots with capacity proportional to the stream.  On the device a call has a
  fixed latency of ~10 us (kernel launch and the first wave) that the CPU reference
  does not see against its ~100 ns per vertex, so the spread is required over the
  counts where the table work dominates (1e6 .. 1e7, the device time of the kernels),
  and the 1e5 point must not cost more device time than the 1e6 one.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _mse(a, b) -> float:
    return float(((a - b) ** 2).mean())


def test_variance_reduction_cornell(gpu):
    from paper_1902_05942_b200.tracer import TraceOptions, trace
    size = 64
    opt = TraceOptions(pixel_jitter=False)
    scene = gpu.load_scene("cornell", size, size)
    ref = trace(scene, 1024, 999, opt).image
    mse = {}
    for jitter in (True, False):
        cfg = gpu.FilterConfig(capacity=1 << (2 * size * size - 1).bit_length(), jitter=jitter)
        r = gpu.run_sequence(scene, cfg, spp=1, seed=1, frames=1, options=opt)[-1]
        mse[jitter] = (_mse(r.filtered, ref), _mse(r.unfiltered, ref))
    filt, unfilt = mse[True]
    assert unfilt >= 3.0 * filt, mse
    assert mse[True][0] <= 1.5 * mse[False][0], mse


def test_constant_time_table_bench(gpu):
    from paper_1902_05942_b200 import bench
    bench.run_point(100_000)  # module / kernel loading
    pts = bench.scaling_sweep((100_000, 1_000_000, 3_000_000, 10_000_000), repeats=3)
    dev = {p.n_vertices: p.device_s for p in pts}
    assert bench.spread(pts[1:], device=True) < 2.0, [p.line() for p in pts]
    assert dev[100_000] <= dev[1_000_000], dev
    # the table is really filled: every vertex landed, ~n/36 cells
    idx, fp, vals = bench.synthetic_stream(1_000_000, 1_000_000 // 36)
    t = gpu.VoxelTable(1 << 20)
    status, slots, _ = t.accumulate_batch(idx, fp, vals, 0)
    assert int((status == 2).sum()) == 0
    assert t.total_counts() == 1_000_000
    assert int((t.lookup_slots(idx, fp) == slots).sum()) == 1_000_000
    torch.cuda.synchronize()
