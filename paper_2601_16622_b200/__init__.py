"""equistream-b200: B200-native (sm_100a) fused on-the-fly equivariant
attention with per-pair EAAS -- the hot path of E2Former-V2 (arXiv
2601.16622) behind the reference `equistream` operator API.

The compute lives in libequistream_b200.so (hand-written CUDA, C ABI in
include/equistream_b200.h).  This package is the Python mirror of the
reference's operator interface (SPEC.md stream_attention / bench modules);
PyTorch only supplies device memory, streams and torch.distributed.
"""
from .api import (  # noqa: F401
    NeighborIndex,
    build_neighbors,
    conventions_manifest,
    neighbors_transpose,
    project_qk,
    project_qk_backward,
    stream_aggregate,
    stream_aggregate_backward,
    tile_mask,
)
from .layer import EquivariantAttention, attention_layer  # noqa: F401

__all__ = [
    "NeighborIndex", "build_neighbors", "neighbors_transpose", "tile_mask", "project_qk", "project_qk_backward",
    "stream_aggregate", "stream_aggregate_backward", "conventions_manifest", "EquivariantAttention",
    "attention_layer",
]
