"""ctypes binding of libequistream_b200.so (the C ABI in include/equistream_b200.h).

There is no CPU fallback: if the library is missing or no sm_100a device is
visible, every compute entry point raises.
"""
from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# ES_LIB_PATH: an experiment build of the same library (A/B variants built with
# ES_NVCC_EXTRA into _variants/); the default is the in-tree build
LIB_PATH = os.environ.get("ES_LIB_PATH") or os.path.join(HERE, "libequistream_b200.so")

ES_OK, ES_INVALID_ARGUMENT, ES_UNSUPPORTED, ES_CUDA_ERROR, ES_NCCL_ERROR = range(5)
ES_F32, ES_BF16 = 0, 1
ES_VALUE_PLAIN, ES_VALUE_EAAS = 0, 1
ES_BIAS_NONE, ES_BIAS_POLY2 = 0, 1
ES_PHI_COSINE, ES_PHI_ONE = 0, 1


class AttnDesc(ct.Structure):
    _fields_ = [("N", ct.c_int32), ("K", ct.c_int32), ("H", ct.c_int32), ("L", ct.c_int32), ("C", ct.c_int32),
                ("value_mode", ct.c_int32), ("phi_mode", ct.c_int32), ("dtype", ct.c_int32),
                ("r_cut", ct.c_double), ("periodic", ct.c_int32), ("box", ct.c_double * 3),
                ("row0", ct.c_int32), ("Nk", ct.c_int32), ("bias_mode", ct.c_int32), ("bias", ct.c_double * 3),
                ("nseg", ct.c_int32)]


ABI_VERSION = 9  # include/equistream_b200.h ES_ABI_VERSION


class NbrDesc(ct.Structure):
    _fields_ = [("N", ct.c_int32), ("K", ct.c_int32), ("nseg", ct.c_int32), ("periodic", ct.c_int32),
                ("r_cut", ct.c_double), ("box", ct.c_double * 3), ("row0", ct.c_int32), ("nrows", ct.c_int32)]


class AttnStats(ct.Structure):
    _fields_ = [(n, ct.c_uint64) for n in ("madds_fwd", "madds_bwd", "madds_proj_fwd", "madds_proj_bwd",
                                           "aux_float_bytes_fwd", "aux_float_bytes_bwd", "aux_index_bytes",
                                           "workspace_fwd_bytes", "workspace_bwd_bytes")]


class TilesSide(ct.Structure):
    _fields_ = [(n, ct.c_int64) for n in ("ntiles", "words", "nchunk_max", "mask", "cptr", "clist", "rowlist",
                                          "tstart", "rtile", "slots", "rank_of")]


class TilesLayout(ct.Structure):
    _fields_ = [("query", TilesSide), ("key", TilesSide)]


class MsgDesc(ct.Structure):
    _fields_ = [("N", ct.c_int32), ("K", ct.c_int32), ("H", ct.c_int32), ("L", ct.c_int32), ("C", ct.c_int32),
                ("origin", ct.c_double * 3)]


class ProjDesc(ct.Structure):
    _fields_ = [("N", ct.c_int32), ("L", ct.c_int32), ("C", ct.c_int32), ("dtype", ct.c_int32)]


class EsError(RuntimeError):
    pass


class EsInvalidArgument(EsError, ValueError):
    """ES_INVALID_ARGUMENT -- the reference's std::invalid_argument."""


class EsUnsupported(EsError):
    pass


_lib = None

EXPORTS = [
    "es_attn_fwd", "es_attn_fwd_workspace_size", "es_attn_tiles_workspace_size", "es_attn_tiles_build", "es_attn_bwd", "es_attn_bwd_workspace_size", "es_neighbors_build",
    "es_neighbors_workspace_size", "es_neighbors_transpose", "es_neighbors_transpose_workspace_size",
    "es_tile_mask", "es_project_fwd", "es_project_bwd", "es_conventions_manifest", "es_cg_real",
    "es_reindex_table", "es_wigner_d_host", "es_last_error", "es_abi_version", "es_device_ok",
    "es_attn_stats_query", "es_attn_tiles_layout_query", "es_translation_coefficients", "es_source_term",
    "es_message_aggregate", "es_target_couple", "es_factorized_workspace_size", "es_factorized_message",
    "es_tp_bench_dense", "es_tp_bench_eaas", "es_tp_madds",
]


def lib() -> ct.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EsError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python -m paper_2601_16622_b200.build); there is no CPU fallback")
        L = ct.CDLL(LIB_PATH)
        vp, i32, sz, dp = ct.c_void_p, ct.c_int32, ct.c_size_t, ct.POINTER(ct.c_double)
        L.es_attn_fwd.argtypes = [ct.POINTER(AttnDesc)] + [vp] * 10 + [sz, vp]
        L.es_attn_tiles_workspace_size.argtypes = [ct.POINTER(AttnDesc)]
        L.es_attn_tiles_workspace_size.restype = sz
        L.es_attn_tiles_build.argtypes = [ct.POINTER(AttnDesc), vp, vp, i32, vp, vp, vp, sz, vp]
        L.es_attn_fwd_workspace_size.argtypes = [ct.POINTER(AttnDesc)]
        L.es_attn_fwd_workspace_size.restype = sz
        L.es_attn_bwd.argtypes = [ct.POINTER(AttnDesc)] + [vp] * 17 + [sz, vp]
        L.es_attn_stats_query.argtypes = [ct.POINTER(AttnDesc), ct.c_int64, ct.POINTER(AttnStats)]
        L.es_attn_tiles_layout_query.argtypes = [ct.POINTER(AttnDesc), ct.POINTER(TilesLayout)]
        md = ct.POINTER(MsgDesc)
        L.es_translation_coefficients.argtypes = [i32, dp]
        L.es_source_term.argtypes = [md, vp, vp, vp, vp]
        L.es_message_aggregate.argtypes = [md, vp, vp, vp, vp, vp]
        L.es_target_couple.argtypes = [md, vp, vp, vp, vp]
        L.es_factorized_workspace_size.argtypes = [md]
        L.es_factorized_workspace_size.restype = sz
        L.es_factorized_message.argtypes = [md, vp, vp, vp, vp, vp, vp, sz, vp]
        L.es_tp_bench_dense.argtypes = [i32, i32, i32, vp, vp, vp, vp]
        L.es_tp_bench_eaas.argtypes = [i32, i32, i32, vp, vp, vp, vp]
        L.es_tp_madds.argtypes = [i32, ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64)]
        L.es_attn_bwd_workspace_size.argtypes = [ct.POINTER(AttnDesc)]
        L.es_attn_bwd_workspace_size.restype = sz
        L.es_neighbors_build.argtypes = [ct.POINTER(NbrDesc)] + [vp] * 6 + [sz, vp]
        L.es_neighbors_workspace_size.argtypes = [ct.POINTER(NbrDesc)]
        L.es_neighbors_workspace_size.restype = sz
        L.es_neighbors_transpose.argtypes = [i32, i32, i32, vp, vp, vp, vp, sz, vp]
        L.es_neighbors_transpose_workspace_size.argtypes = [i32, i32, i32]
        L.es_neighbors_transpose_workspace_size.restype = sz
        L.es_tile_mask.argtypes = [i32, i32, vp, i32, i32, vp, vp]
        L.es_project_fwd.argtypes = [ct.POINTER(ProjDesc)] + [vp] * 6
        L.es_project_bwd.argtypes = [ct.POINTER(ProjDesc)] + [vp] * 8
        L.es_conventions_manifest.restype = ct.c_char_p
        L.es_last_error.restype = ct.c_char_p
        L.es_cg_real.restype = ct.c_double
        L.es_cg_real.argtypes = [i32] * 6
        L.es_reindex_table.argtypes = [i32, i32, i32, i32, dp, dp]
        L.es_wigner_d_host.argtypes = [i32, dp, dp]
        if L.es_abi_version() != ABI_VERSION:
            raise EsError("libequistream_b200.so ABI mismatch: rebuild (python -m paper_2601_16622_b200.build)")
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status == ES_OK:
        return
    msg = f"{what}: {lib().es_last_error().decode(errors='replace')}"
    if status == ES_INVALID_ARGUMENT:
        raise EsInvalidArgument(msg)
    if status == ES_UNSUPPORTED:
        raise EsUnsupported(msg)
    raise EsError(msg)
