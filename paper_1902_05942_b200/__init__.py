"""B200-native hashed path-space filtering (arXiv 1902.05942).

Drop-in for the reference package `pathfilter` (src/__init__.py:10-33): build keys,
insert vertices, query averages, temporal update -- plus the on-device path tracer
that produces the vertex stream, whole frames (render_frame / run_sequence, all three
temporal modes) and the key-sharded multi-GPU frame.  All compute runs in hand-written
sm_100a CUDA kernels (libpf_b200.so, C ABI in include/pathfilter_b200.h); there is no
CPU fallback.  The reference's one-vertex-at-a-time scalar key helpers and brute-force
partition utilities (src/keys.py:104-240, src/oracle.py) are not part of this package:
the batched key path (make_key_arrays / vertex_keys) is the filter API, and the CPU
restatement used as a checker lives in oracle/ (test infrastructure).
"""

from . import rng
from .images import read_ppm, tonemap, write_ppm
from .keys import CellHashes, CellKey, FilterConfig, KeyArrays, hash_arrays, hashes, \
    make_key_arrays, pack_aux
from .pipeline import FrameState, FrameStats, ResolveReport, VertexStream, accumulate_phase, \
    filter_frame, resolve_phase, vertex_keys
from .render import FrameResult, render_frame, run_sequence
from .scene import Camera, Material, Motion, Scene, SceneBuilder, SceneError, closed_box, \
    cornell_box, load_scene, parse_scene
from .table import EMPTY_TAG, EvictionEvent, InsertOutcome, Outcome, VoxelTable, \
    fixed_to_float, pack_priority, quantize_fixed
from .temporal import migrate_cells, migrate_resolution, reevaluation_deltas, \
    select_replay_ids
from .tracer import TraceOptions, TraceResult, reevaluate, trace

from ._backend import BACKEND, available_backends
from .keys import aux_bits_array, jittered_positions, levels_array, normal_bins_array, \
    tangent_basis_array
from .host import HostFrame, HostFramePipeline
from .pipeline import VertexDescriptor

__version__ = "0.1.0"


__all__ = [
    "BACKEND", "available_backends", "rng", "CellHashes", "CellKey", "FilterConfig",
    "KeyArrays", "hash_arrays", "hashes", "make_key_arrays", "pack_aux", "FrameState", "FrameStats", "ResolveReport",
    "VertexStream", "accumulate_phase", "filter_frame", "resolve_phase", "vertex_keys",
    "FrameResult", "render_frame", "run_sequence", "Camera", "Material", "Motion", "Scene",
    "SceneBuilder", "SceneError", "closed_box", "cornell_box", "load_scene", "parse_scene",
    "EMPTY_TAG", "EvictionEvent", "InsertOutcome", "Outcome", "VoxelTable", "fixed_to_float",
    "pack_priority", "quantize_fixed", "migrate_cells", "migrate_resolution",
    "reevaluation_deltas", "select_replay_ids", "TraceOptions", "TraceResult", "reevaluate",
    "trace", "read_ppm", "tonemap", "write_ppm", "VertexDescriptor", "levels_array",
    "tangent_basis_array", "jittered_positions", "normal_bins_array", "aux_bits_array",
    "HostFrame", "HostFramePipeline",
]
