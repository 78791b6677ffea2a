"""Python mirror of the reference operator interface for the hot path
(SPEC.md stream_attention :232-325, bench.build_neighbors :431-439), over the
C ABI.  Names, argument meaning and error behaviour follow the SPEC:
shape/precondition violations raise ValueError (EsInvalidArgument, the
reference's std::invalid_argument), internal/CUDA failures RuntimeError.

All tensors are CUDA tensors; launches go to torch's current stream.  No
CPU fallback exists -- a CPU tensor is an argument error.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import EsInvalidArgument, check, lib

_DT = {torch.float32: _lib.ES_F32, torch.bfloat16: _lib.ES_BF16}
_VALUE = {"plain": _lib.ES_VALUE_PLAIN, "eaas": _lib.ES_VALUE_EAAS}
_PHI = {"cosine": _lib.ES_PHI_COSINE, "one": _lib.ES_PHI_ONE}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, name: str, dtype=None, shape=None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise EsInvalidArgument(f"{name}: expected a tensor")
    if not t.is_cuda:
        raise EsInvalidArgument(f"{name}: must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise EsInvalidArgument(f"{name}: dtype {t.dtype}, expected {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise EsInvalidArgument(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise EsInvalidArgument(f"{name}: must be contiguous")
    return t


def aligned_positions(pos: torch.Tensor) -> torch.Tensor:
    """pos, or a 16-byte-aligned copy of it (a view such as pos[a0:a1] with
    odd a0 is only 8-byte aligned; es_attn_fwd requires 16)."""
    return pos if pos.data_ptr() % 16 == 0 and pos.is_contiguous() else pos.contiguous().clone()


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def wigner_d(l: int, R) -> "np.ndarray":
    """D^l(R) [(2l+1)][(2l+1)] acting on value vectors (solid(l, R r) =
    D solid(l, r)), from the library's host tables (es_wigner_d_host)."""
    import numpy as np
    Rm = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
    D = np.zeros((2 * l + 1) ** 2)
    check(lib().es_wigner_d_host(int(l), Rm.ctypes.data_as(ct.POINTER(ct.c_double)),
                                 D.ctypes.data_as(ct.POINTER(ct.c_double))), "es_wigner_d_host")
    return D.reshape(2 * l + 1, 2 * l + 1)


def rotate_features(x: torch.Tensor, L: int, R) -> torch.Tensor:
    """rotate_feature (irreps.hpp:104-112) for the [N][M][C] layout: every
    degree block's value vectors v -> D^l(R) v."""
    out = torch.empty_like(x)
    wd = torch.float64 if x.dtype == torch.float64 else torch.float32
    for l in range(L + 1):
        D = torch.tensor(wigner_d(l, R), dtype=wd, device=x.device)
        blk = x[:, l * l:(l + 1) ** 2, :].to(wd)
        out[:, l * l:(l + 1) ** 2, :] = torch.einsum("ab,nbc->nac", D, blk).to(x.dtype)
    return out


def conventions_manifest() -> str:
    return lib().es_conventions_manifest().decode()


# ------------------------------------------------------------------ neighbours
@dataclass
class NeighborIndex:
    """NeighborIndex: table [N][K] int32, sentinel -1,
    rows sorted by (d^2, j); distances [N][K] float32; count [N]."""
    table: torch.Tensor
    distances: torch.Tensor | None
    count: torch.Tensor
    r_cut: float
    box: tuple | None = None
    _rev: tuple | None = None
    seg_ptr: torch.Tensor | None = None  # molecule segments the index was built with (packed query tiles)

    @property
    def N(self) -> int:
        return self.table.shape[0]

    @property
    def K(self) -> int:
        return self.table.shape[1]

    @property
    def nseg(self) -> int:
        return 0 if self.seg_ptr is None else int(self.seg_ptr.numel()) - 1

    def tiles(self, d: "_lib.AttnDesc") -> torch.Tensor | None:
        """The tile structures (tile-skip mask, chunk lists, per-row chunk
        masks and slot order) the tensor-core kernels walk for this index --
        built once (es_attn_tiles_build) and reused by every forward /
        backward / layer on it; None when the kernels for `d` need none."""
        nbytes = lib().es_attn_tiles_workspace_size(ct.byref(d))
        if nbytes == 0:
            return None
        key = (d.N, d.K, d.Nk, d.row0, nbytes)
        cache = self.__dict__.setdefault("_tiles", {})
        if key not in cache:
            buf = torch.empty(int(nbytes), dtype=torch.uint8, device=self.table.device)
            seg = self.seg_ptr if (self.seg_ptr is not None and d.row0 == 0 and d.N == self.N) else None
            nseg = 0 if seg is None else seg.numel() - 1
            rev_ptr, rev_pair = self.transpose(d.Nk if d.Nk > 0 else self.N)  # key-side lists of the backward
            check(lib().es_attn_tiles_build(ct.byref(d), _ptr(self.table), _ptr(seg), nseg, _ptr(rev_ptr),
                                            _ptr(rev_pair), _ptr(buf), buf.numel(), _stream()),
                  "es_attn_tiles_build")
            cache[key] = buf
        return cache[key]

    def transpose(self, n_keys: int | None = None):
        nk = self.N if n_keys is None else int(n_keys)
        if self._rev is None or self._rev[0].numel() != nk + 1:
            self._rev = neighbors_transpose(self.table, nk)
        return self._rev


def build_neighbors(pos: torch.Tensor, K: int, r_cut: float, seg_ptr: torch.Tensor | None = None,
                    box=None, with_distances: bool = True, rows: tuple[int, int] | None = None) -> NeighborIndex:
    """build_neighbors: K nearest j != i with |r_ij| < r_cut,
    inside the atom's segment (molecule batch) and under the minimum image
    when `box` is given.  Bit-identical to the CPU oracle.  rows=(a0, a1):
    only query rows a0..a1-1 (a row shard; keys are all atoms) -- the
    returned index holds a1 - a0 rows with global key ids."""
    pos = _need(pos, "pos", torch.float64)
    if pos.dim() != 2 or pos.shape[1] != 3:
        raise EsInvalidArgument("pos: expected [N, 3]")
    if K < 1:
        raise EsInvalidArgument("build_neighbors: K >= 1")
    N = pos.shape[0]
    dev = pos.device
    d = _lib.NbrDesc()
    d.N, d.K, d.r_cut = N, int(K), float(r_cut)
    d.nseg = 0
    if seg_ptr is not None:
        seg_ptr = _need(seg_ptr, "seg_ptr", torch.int32)
        d.nseg = seg_ptr.numel() - 1
    d.periodic = 0 if box is None else 1
    if box is not None:
        for a in range(3):
            d.box[a] = float(box[a])
    nr = N
    if rows is not None:
        a0, a1 = int(rows[0]), int(rows[1])
        if not 0 <= a0 <= a1 <= N:
            raise EsInvalidArgument("build_neighbors: rows must satisfy 0 <= a0 <= a1 <= N")
        nr = a1 - a0
        d.row0, d.nrows = (a0, nr) if nr > 0 else (0, 0)
    nbr = torch.empty((nr, K), dtype=torch.int32, device=dev)
    dist = torch.empty((nr, K), dtype=torch.float32, device=dev) if with_distances else None
    cnt = torch.empty((nr,), dtype=torch.int32, device=dev)
    if nr == 0:
        return NeighborIndex(nbr, dist, cnt, float(r_cut), None if box is None else tuple(float(b) for b in box))
    ws = _workspace(lib().es_neighbors_workspace_size(ct.byref(d)), dev)
    check(lib().es_neighbors_build(ct.byref(d), _ptr(pos), _ptr(seg_ptr), _ptr(nbr), _ptr(dist), _ptr(cnt),
                                   _ptr(ws), ws.numel(), _stream()), "es_neighbors_build")
    return NeighborIndex(nbr, dist, cnt, float(r_cut), None if box is None else tuple(float(b) for b in box),
                         seg_ptr=seg_ptr if rows is None else None)


def neighbors_transpose(table: torch.Tensor, n_keys: int | None = None):
    """Key-major relation over n_keys key atoms (default N): (rev_ptr [Nk+1],
    rev_pair [N*K]) with rev_pair[rev_ptr[j]:rev_ptr[j+1]] = sorted
    {i*K+slot : table[i,slot] == j}."""
    table = _need(table, "table", torch.int32)
    N, K = table.shape
    Nk = N if n_keys is None else int(n_keys)
    rev_ptr = torch.empty(Nk + 1, dtype=torch.int32, device=table.device)
    rev_pair = torch.empty(max(N * K, 1), dtype=torch.int32, device=table.device)
    ws = _workspace(lib().es_neighbors_transpose_workspace_size(N, K, Nk), table.device)
    check(lib().es_neighbors_transpose(N, K, Nk, _ptr(table), _ptr(rev_ptr), _ptr(rev_pair), _ptr(ws), ws.numel(),
                                       _stream()), "es_neighbors_transpose")
    return rev_ptr, rev_pair


def tile_mask(table: torch.Tensor, tq: int = 32, tk: int = 32) -> torch.Tensor:
    """Tile-skip bitmask [ceil(N/tq)][ceil(ceil(N/tk)/32)] uint32 (stored int32)."""
    table = _need(table, "table", torch.int32)
    N, K = table.shape
    nqb = (N + tq - 1) // tq
    words = ((N + tk - 1) // tk + 31) // 32
    mask = torch.zeros((nqb, words), dtype=torch.int32, device=table.device)
    check(lib().es_tile_mask(N, K, _ptr(table), tq, tk, _ptr(mask), _stream()), "es_tile_mask")
    return mask


# ------------------------------------------------------------------ projections
def _proj_desc(h: torch.Tensor, L: int) -> _lib.ProjDesc:
    d = _lib.ProjDesc()
    d.N, d.L, d.C = h.shape[0], int(L), h.shape[2]
    d.dtype = _DT[h.dtype]
    return d


def project_qk(h: torch.Tensor, W: torch.Tensor, L: int):
    """project_qk + W_H (Eq. 6): h [N][M][C], W [L+1][C][5C]
    -> q, k [N][M][2C], v [N][M][C] (same dtype)."""
    if h.dtype not in _DT:
        raise EsInvalidArgument("h: dtype must be float32 or bfloat16")
    M = (L + 1) ** 2
    _need(h, "h")
    if h.dim() != 3 or h.shape[1] != M:
        raise EsInvalidArgument(f"h: expected [N, {M}, C]")
    N, _, C = h.shape
    _need(W, "W", h.dtype, (L + 1, C, 5 * C))
    q = torch.empty((N, M, 2 * C), dtype=h.dtype, device=h.device)
    k = torch.empty_like(q)
    v = torch.empty((N, M, C), dtype=h.dtype, device=h.device)
    d = _proj_desc(h, L)
    check(lib().es_project_fwd(ct.byref(d), _ptr(h), _ptr(W), _ptr(q), _ptr(k), _ptr(v), _stream()),
          "es_project_fwd")
    return q, k, v


def project_qk_backward(h, W, L, dq, dk, dv, want_dW: bool = True):
    d = _proj_desc(h, L)
    for t, n in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        _need(t, n, h.dtype)
    dh = torch.empty_like(h)
    dW = torch.empty(W.shape, dtype=torch.float32, device=h.device) if want_dW else None
    check(lib().es_project_bwd(ct.byref(d), _ptr(h), _ptr(W), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dh), _ptr(dW),
                               _stream()), "es_project_bwd")
    return dh, dW


# ------------------------------------------------------------------ attention
@dataclass
class AttentionConfig:
    heads: int
    L: int
    r_cut: float = 6.0
    value_mode: str = "eaas"
    phi: str = "cosine"
    box: tuple | None = None
    bias: tuple | None = None  # radial score bias b(r) = b0 + b1 r + b2 r^2 (None: b == 0)
    keep_scores: bool = False  # the forward keeps the O(N K H) scores for the backward (pays with ES_DK_TC=1)

    def desc(self, N: int, K: int, C: int, dtype: torch.dtype, row0: int = 0, Nk: int = 0,
             nseg: int = 0) -> _lib.AttnDesc:
        if self.value_mode not in _VALUE:
            raise EsInvalidArgument(f"value_mode must be one of {list(_VALUE)}")
        if self.phi not in _PHI:
            raise EsInvalidArgument(f"phi must be one of {list(_PHI)}")
        d = _lib.AttnDesc()
        d.N, d.K, d.H, d.L, d.C = N, K, int(self.heads), int(self.L), C
        d.value_mode = _VALUE[self.value_mode]
        d.phi_mode = _PHI[self.phi]
        d.dtype = _DT[dtype]
        d.r_cut = float(self.r_cut)
        d.nseg = int(nseg)
        if self.bias is not None:
            b = tuple(float(x) for x in self.bias) + (0.0,) * (3 - len(self.bias))
            d.bias_mode = _lib.ES_BIAS_POLY2
            for a in range(3):
                d.bias[a] = b[a]
        d.periodic = 0 if self.box is None else 1
        if self.box is not None:
            for a in range(3):
                d.box[a] = float(self.box[a])
        d.row0, d.Nk = int(row0), int(Nk)
        return d


@dataclass
class SavedAttention:
    """What stream_aggregate_backward needs (SPEC.md:293 'saved inputs')."""
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    pos: torch.Tensor
    idx: NeighborIndex
    out: torch.Tensor
    lse: torch.Tensor
    cfg: AttentionConfig
    row0: int = 0
    scores: torch.Tensor | None = None  # the forward's [N][K][H] scores (optional)


def _check_qkv(q, k, v, pos, idx, cfg, row0=0):
    """q (and idx, out, lse): the N local query rows; k, v, pos: all Nk atoms."""
    if q.dtype not in _DT:
        raise EsInvalidArgument("q: dtype must be float32 or bfloat16")
    M = (cfg.L + 1) ** 2
    _need(v, "v", q.dtype)
    if v.dim() != 3 or v.shape[1] != M:
        raise EsInvalidArgument(f"v: expected [Nk, {M}, C]")
    Nk, _, C = v.shape
    _need(q, "q", q.dtype)
    if q.dim() != 3 or tuple(q.shape[1:]) != (M, 2 * C):
        raise EsInvalidArgument(f"q: expected [N, {M}, {2 * C}]")
    N = q.shape[0]
    _need(k, "k", q.dtype, (Nk, M, 2 * C))
    _need(pos, "pos", torch.float64, (Nk, 3))
    if pos.data_ptr() % 16:
        raise EsInvalidArgument("pos: must be 16-byte aligned (use aligned_positions())")
    _need(idx.table, "idx.table", torch.int32)
    if idx.table.shape[0] != N:
        raise EsInvalidArgument("idx: row count != number of query rows")
    if row0 < 0 or row0 + N > Nk:
        raise EsInvalidArgument("row0 + N > Nk")
    return N, C, Nk


def stream_aggregate(q, k, v, pos, idx: NeighborIndex, cfg: AttentionConfig, row0: int = 0,
                     return_scores: bool = False):
    """stream_aggregate (Alg. 1): returns (m [N][M][C], lse [N][H] f32)
    -- plus the [H][N][K] scores with return_scores (a row's valid scores in its
    first count entries, in a library-private order; pass them back to
    stream_aggregate_backward through SavedAttention.scores).
    With row0 / k, v, pos longer than q: the query rows are atoms row0..row0+N-1
    of the Nk-atom system (query-row sharding)."""
    N, C, Nk = _check_qkv(q, k, v, pos, idx, cfg, row0)
    out = torch.empty((N,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
    lse = torch.empty((N, cfg.heads), dtype=torch.float32, device=v.device)
    scores = torch.empty((cfg.heads, N, idx.K), dtype=torch.float32, device=v.device) if return_scores else None
    d = cfg.desc(N, idx.K, C, q.dtype, row0, Nk, idx.nseg if row0 == 0 and Nk == N else 0)
    tiles = idx.tiles(d)
    ws = _workspace(256 if tiles is not None else lib().es_attn_fwd_workspace_size(ct.byref(d)), q.device)
    check(lib().es_attn_fwd(ct.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(pos), _ptr(idx.table), _ptr(out),
                            _ptr(lse), _ptr(scores), _ptr(tiles), _ptr(ws), ws.numel(), _stream()), "es_attn_fwd")
    if return_scores:
        return out, lse, scores
    return out, lse


def attn_stats(cfg: AttentionConfig, N: int, K: int, C: int, n_pairs: int, dtype=torch.bfloat16, Nk: int = 0):
    """OpCounters / stats structure (counters.hpp:11-32):
    algorithmic multiply-adds and the auxiliary device memory of one layer."""
    d = cfg.desc(N, K, C, dtype, 0, Nk)
    st = _lib.AttnStats()
    check(lib().es_attn_stats_query(ct.byref(d), int(n_pairs), ct.byref(st)), "es_attn_stats_query")
    return {n: int(getattr(st, n)) for n, _ in st._fields_}


def stream_aggregate_backward(grad_m: torch.Tensor, saved: SavedAttention, pos_grad: bool = False):
    """stream_aggregate_backward: (grad_q, grad_k, grad_v) of
    sum <grad_m, m>, by recomputation (no O(N*K*C) buffer).  pos_grad=True
    (any L) also returns grad_pos [Nk][3] f64 -- the position gradient through
    phi(r_ij) and the solid harmonics of the value map (forces):
    (grad_q, grad_k, grad_v, grad_pos)."""
    s = saved
    N, C, Nk = _check_qkv(s.q, s.k, s.v, s.pos, s.idx, s.cfg, s.row0)
    grad_m = _need(grad_m.contiguous(), "grad_m", s.q.dtype, tuple(s.out.shape))
    rev_ptr, rev_pair = s.idx.transpose(Nk)
    d = s.cfg.desc(N, s.idx.K, C, s.q.dtype, s.row0, Nk, s.idx.nseg if s.row0 == 0 and Nk == N else 0)
    ws = _workspace(lib().es_attn_bwd_workspace_size(ct.byref(d)), s.q.device)
    dq = torch.empty_like(s.q)
    dk = torch.empty_like(s.k)
    dv = torch.empty_like(s.v)
    dpos = torch.empty((Nk, 3), dtype=torch.float64, device=s.q.device) if pos_grad else None
    tiles = s.idx.tiles(d)
    check(lib().es_attn_bwd(ct.byref(d), _ptr(s.q), _ptr(s.k), _ptr(s.v), _ptr(s.pos), _ptr(s.idx.table),
                            _ptr(rev_ptr), _ptr(rev_pair), _ptr(s.out), _ptr(s.lse), _ptr(s.scores), _ptr(grad_m),
                            _ptr(dq),
                            _ptr(dk), _ptr(dv), _ptr(dpos), _ptr(tiles), _ptr(ws), ws.numel(), _stream()),
          "es_attn_bwd")
    return (dq, dk, dv, dpos) if pos_grad else (dq, dk, dv)


# ------------------------------------------------------------------ factorized message
def translation_coefficients(l: int):
    """translation_coefficients: w[u] of R^l(a+b) = sum_u w[u] (R^u(a) x R^{l-u}(b))^l."""
    import numpy as np
    w = np.zeros(l + 1)
    check(lib().es_translation_coefficients(int(l), w.ctypes.data_as(ct.POINTER(ct.c_double))),
          "es_translation_coefficients")
    return w


def _msg_desc(pos, h, K, H, L, origin):
    d = _lib.MsgDesc()
    d.N, d.K, d.H, d.L, d.C = h.shape[0], int(K), int(H), int(L), h.shape[2]
    o = pos.mean(dim=0).tolist() if origin is None else [float(x) for x in origin]
    for a in range(3):
        d.origin[a] = o[a]
    return d


def factorized_message(pos: torch.Tensor, h: torch.Tensor, nbr: torch.Tensor, alpha: torch.Tensor, L: int,
                       origin=None, stages: bool = False):
    """factorized_message (Eq. 5): source_term -> alpha
    aggregation -> target_couple on the GPU in fp64.  pos [N,3], h [N,M,C],
    nbr [N,K] int32, alpha [N,K,H] (all float64 except nbr); origin defaults
    to the centroid (the SPEC's recentring).  stages=True also returns the
    source terms S and aggregates A ([N, (L+1)^4, C])."""
    _need(pos, "pos", torch.float64)
    _need(h, "h", torch.float64)
    _need(nbr, "nbr", torch.int32)
    _need(alpha, "alpha", torch.float64)
    N, K = nbr.shape
    H = alpha.shape[2]
    d = _msg_desc(pos, h, K, H, L, origin)
    out = torch.empty_like(h)
    if stages:
        S = torch.empty((N, (L + 1) ** 4, h.shape[2]), dtype=torch.float64, device=h.device)
        A = torch.empty_like(S)
        check(lib().es_source_term(ct.byref(d), _ptr(pos), _ptr(h), _ptr(S), _stream()), "es_source_term")
        check(lib().es_message_aggregate(ct.byref(d), _ptr(nbr), _ptr(alpha), _ptr(S), _ptr(A), _stream()),
              "es_message_aggregate")
        check(lib().es_target_couple(ct.byref(d), _ptr(pos), _ptr(A), _ptr(out), _stream()), "es_target_couple")
        return out, S, A
    ws = _workspace(lib().es_factorized_workspace_size(ct.byref(d)), h.device)
    check(lib().es_factorized_message(ct.byref(d), _ptr(pos), _ptr(h), _ptr(nbr), _ptr(alpha), _ptr(out), _ptr(ws),
                                      ws.numel(), _stream()), "es_factorized_message")
    return out


# ------------------------------------------------------------------ tensor-product microbenchmark
def tp_madds(L: int):
    """(dense, EAAS) multiply-adds per pair-channel of the path-set product (run_tp_bench)."""
    a, b = ct.c_int64(), ct.c_int64()
    check(lib().es_tp_madds(int(L), ct.byref(a), ct.byref(b)), "es_tp_madds")
    return a.value, b.value


def tensor_product_pairs(v: torch.Tensor, r: torch.Tensor, L: int, method: str = "eaas") -> torch.Tensor:
    """x_p = sum_paths (v_p^li (x) R^lf(r_p))^lo for P independent pairs, by the dense
    CG product or by EAAS (the fused kernels' per-pair device code); f32."""
    _need(v, "v", torch.float32)
    _need(r, "r", torch.float32, (v.shape[0], 3))
    x = torch.empty_like(v)
    fn = lib().es_tp_bench_eaas if method == "eaas" else lib().es_tp_bench_dense
    check(fn(int(L), v.shape[2], v.shape[0], _ptr(v), _ptr(r), _ptr(x), _stream()), f"es_tp_bench_{method}")
    return x
