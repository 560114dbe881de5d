"""The kernel-module drop-in (src/_backend.py:14-42 -> paper_1902_05942_b200.kernels)
driven by the REFERENCE's own VoxelTable and tests.

- the reference's pkg/tests/test_table.py, unmodified, with its backend routed to the
  device module (tests/dropin_plugin.py), including its multi-threaded cases;
- several threads inserting into one host table: no lost counts or sums;
- host-side mutations between calls (begin_frame) are seen by the next call;
- a 10^6-vertex batch into C = 2^22 tables: same per-key contents as the reference's
  native Cython kernel, and faster than it."""

import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "_ref_tests")
need_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "pathfilter")),
                              reason="baseline/_ref absent (tools/install_reference.sh)")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import pathfilter
    from pathfilter import table
    return pathfilter, table


def _canon(t):
    """Order-free table contents: occupied rows sorted on every column."""
    occ = np.nonzero(t.tags != np.uint64(0xFFFFFFFF00000000))[0]
    cols = [t.tags[occ].view(np.int64), t.counts[occ], t.hist_counts[occ], t.last_touch[occ]]
    cols += [t.sums[occ, c].view(np.int64) for c in range(3)]
    cols += [t.hist_sums[occ, c].view(np.int64) for c in range(3)]
    m = np.stack(cols, axis=1)
    return m[np.lexsort(m.T[::-1])]


@need_ref
@pytest.mark.skipif(not os.path.exists(os.path.join(REF_TESTS, "test_table.py")),
                    reason="reference tests not staged (tools/install_reference.sh)")
def test_reference_table_suite_on_device_kernels(gpu, tmp_path):
    report = tmp_path / "calls.json"
    env = dict(os.environ, PF_DROPIN_REPORT=str(report),
               PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT]))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin",
                          "-p", "no:cacheprovider", "--rootdir", REF_TESTS,
                          os.path.join(REF_TESTS, "test_table.py")],
                         capture_output=True, text=True, timeout=900, cwd=REF_TESTS, env=env)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and "failed" not in out.stdout, tail
    rep = json.loads(report.read_text())
    assert rep["backend"] == "b200"
    assert rep["calls"]["accumulate_fixed"] > 20 and rep["calls"]["lookup_slots"] > 5, rep


@need_ref
@pytest.mark.parametrize("sum_mode", ["fixed", "float"])
def test_threads_on_one_host_table_lose_nothing(gpu, sum_mode):
    """concurrent accumulate calls on one numpy table.  8 threads x
    20 batches of 5000 vertices (parallel kernel) over 3000 keys: every count and
    (fixed mode) every fixed-point sum arrives."""
    from paper_1902_05942_b200 import kernels
    pf, table = _ref()
    t = table.VoxelTable(1 << 16, sum_mode=sum_mode)
    fn = kernels.accumulate_fixed if sum_mode == "fixed" else kernels.accumulate_float
    r = np.random.default_rng(3)
    keys = r.integers(0, 2**63, 3000).astype(np.uint64)
    batches = []
    for _ in range(8 * 20):
        k = keys[r.integers(0, len(keys), 5000)]
        batches.append((k, (k >> np.uint64(17)).astype(np.uint32) | np.uint32(1),
                        r.uniform(0, 2, (5000, 3))))
    errors = []

    def worker(w):
        try:
            for b in batches[w::8]:
                fn(t.tags, t.sums, t.counts, t.hist_sums, t.hist_counts, t.last_touch,
                   t.deltas, b[0], b[1], b[2], 0, t.probe_limit, t.evict_min_age)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=worker, args=(w,)) for w in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    assert int(t.counts.sum()) == 8 * 20 * 5000
    vals = np.concatenate([b[2] for b in batches])
    if sum_mode == "fixed":
        want = table.quantize_fixed(vals).sum(axis=0)
        assert np.array_equal(t.sums.sum(axis=0), want)
    else:
        np.testing.assert_allclose(t.sums.sum(axis=0), vals.sum(axis=0), rtol=1e-9)


@need_ref
def test_host_mutations_between_calls_are_seen(gpu):
    """The host table stays authoritative: the reference's own begin_frame (numpy, on
    the host) between device calls; every frame equals the native kernel's table."""
    pf, table = _ref()
    from pathfilter import _native
    from paper_1902_05942_b200 import kernels
    cfg = pf.FilterConfig(capacity=1 << 11, temporal_mode="filter")
    a = table.VoxelTable(cfg.capacity, cfg.probe_limit, "fixed", 4, 1)
    b = table.VoxelTable(cfg.capacity, cfg.probe_limit, "fixed", 4, 1)
    a._k, b._k = _native, kernels
    r = np.random.default_rng(9)
    keys = r.integers(0, 2**63, 4000).astype(np.uint64)
    for f in range(8):
        a.begin_frame(f, cfg)
        b.begin_frame(f, cfg)
        k = keys[r.integers(f * 300, f * 300 + 900, 3000)]   # drifting key set: evictions
        fp = (k >> np.uint64(11)).astype(np.uint32) | np.uint32(1)
        v = r.uniform(0, 1, (3000, 3))
        ra = a.accumulate_batch(k, fp, v, f)
        rb = b.accumulate_batch(k, fp, v, f)
        for x, y in zip(ra, rb):   # < 4096 vertices: the sequential order, bit for bit
            assert np.array_equal(x, y), f
        for name in ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch",
                     "deltas"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), (f, name)
        assert len(a.eviction_events) == len(b.eviction_events)
    assert len(a.eviction_events) > 0 and a.horizon_clears > 0


@need_ref
def test_million_vertex_batch_matches_native_and_is_faster(gpu):
    pf, table = _ref()
    from pathfilter import _native
    from paper_1902_05942_b200 import kernels
    cap, n = 1 << 22, 1_000_000
    r = np.random.default_rng(1)
    keys = r.integers(0, 2**63, 60_000).astype(np.uint64)
    a = table.VoxelTable(cap)
    b = table.VoxelTable(cap)
    a._k, b._k = _native, kernels
    fp_of = lambda k: (k >> np.uint64(13)).astype(np.uint32) | np.uint32(1)  # noqa: E731
    # one warm-up batch of the same size each: first touch of the host pages, the device
    # mirror and its page-locking, the parallel kernel's lazy module load
    w = keys[r.integers(0, len(keys), n)]
    wv = r.uniform(0, 4, (n, 3))
    for t in (a, b):
        t.accumulate_batch(w, fp_of(w), wv, 0)
    k = keys[r.integers(0, len(keys), n)]
    fp = fp_of(k)
    v = r.uniform(0, 4, (n, 3))
    t0 = time.perf_counter()
    a.accumulate_batch(k, fp, v, 0)
    t_native = time.perf_counter() - t0
    t0 = time.perf_counter()
    b.accumulate_batch(k, fp, v, 0)
    t_dev = time.perf_counter() - t0
    assert np.array_equal(_canon(a), _canon(b))
    assert int(a.counts.sum()) == int(b.counts.sum()) == 2 * n
    print(f"1e6-vertex batch at C=2^22: native {t_native * 1e3:.1f} ms, "
          f"b200 drop-in {t_dev * 1e3:.1f} ms")
    assert t_dev < t_native
