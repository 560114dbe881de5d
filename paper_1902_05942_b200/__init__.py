"""B200-native hashed path-space filtering (arXiv 1902.05942).

Drop-in for the filter API of the reference package `pathfilter`
(src/__init__.py:10-33): build keys, insert vertices, query averages, temporal
update.  All compute runs in hand-written sm_100a CUDA kernels
(libpf_b200.so, C ABI in include/pathfilter_b200.h); there is no CPU fallback.
"""

from . import rng
from .keys import CellHashes, CellKey, FilterConfig, KeyArrays, hash_arrays, hashes, \
    make_key_arrays, pack_aux
from .pipeline import FrameState, FrameStats, ResolveReport, VertexStream, accumulate_phase, \
    filter_frame, resolve_phase, vertex_keys
from .table import EMPTY_TAG, EvictionEvent, InsertOutcome, Outcome, VoxelTable, \
    fixed_to_float, pack_priority, quantize_fixed

BACKEND = "b200"
__version__ = "0.1.0"

__all__ = [
    "BACKEND", "rng", "CellHashes", "CellKey", "FilterConfig", "KeyArrays", "hash_arrays",
    "hashes", "make_key_arrays", "pack_aux", "FrameState", "FrameStats", "ResolveReport",
    "VertexStream", "accumulate_phase", "filter_frame", "resolve_phase", "vertex_keys",
    "EMPTY_TAG", "EvictionEvent", "InsertOutcome", "Outcome", "VoxelTable", "fixed_to_float",
    "pack_priority", "quantize_fixed",
]
