"""Counter-based RNG constants and the host-side seed schedule (src/rng.py).

Per-vertex draws run on the device (csrc/pf_device.cuh: jitter_draws).  The host
only folds the seed and stream tag into the 64-bit stream base once per call
(src/rng.py:68) and derives per-frame seeds (src/pipeline.py:329).
"""

from __future__ import annotations

MASK64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xFF51AFD7ED558CCD
_M2 = 0xC4CEB9FE1A85EC53

STREAM_TRACE = 1          # src/rng.py:19
STREAM_JITTER_ACCUM = 2   # src/rng.py:20
STREAM_JITTER_LOOKUP = 3  # src/rng.py:21


def mix64(x: int) -> int:
    """murmur3 fmix64 (src/rng.py:26-34) on one host integer."""
    x &= MASK64
    x ^= x >> 33
    x = (x * _M1) & MASK64
    x ^= x >> 33
    x = (x * _M2) & MASK64
    x ^= x >> 33
    return x


def stream_base(seed: int, stream: int) -> int:
    """h0 = mix64(seed ^ stream*G): the per-call constant of draw_u64_array (src/rng.py:68)."""
    return mix64((int(seed) & MASK64) ^ ((int(stream) * GOLDEN) & MASK64))


def frame_seed(seed: int, frame: int) -> int:
    """Per-frame seed of animated scenes (src/pipeline.py:329)."""
    return mix64(int(seed) ^ (int(frame) * GOLDEN))
