"""Multi-GPU execution of the hot path (SURVEY.md §8 e): one process per GPU
(torchrun), torch.distributed over NCCL / NVLink for the plumbing.

Two ways the path shards, and only those (no invented collectives):

* Molecule batches (configs 2, 4): molecules are independent, so
  `shard_molecules` hands every rank a contiguous, atom-balanced range of
  whole molecules; forward and backward need no data-path collective (the
  weight gradient is summed with one all-reduce of ~1 MB if requested).

* One large system (config 5): `RowShardedAttention` partitions the query
  rows into contiguous slabs.  Each rank projects its own atoms, all-gathers
  K and V once per layer (positions are a replicated input), runs the fused
  attention for its rows against all keys (the ABI's row0 / Nk), and in the
  backward keeps dq local while the partial dk / dv of all keys are
  reduce-scattered to their owners.

The per-GPU compute goes through `backend` (default: the CUDA library via
paper_2601_16622_b200.api).  Tests substitute a CPU oracle backend to check
the sharding and collective wiring with gloo; the product path has no CPU
fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


# ------------------------------------------------------------------ molecules
def shard_molecules(seg_ptr, world: int, rank: int):
    """Contiguous molecule range [m0, m1) of `rank`, balanced by atom count.
    Returns (m0, m1, a0, a1, local_seg_ptr)."""
    seg = np.asarray(seg_ptr, dtype=np.int64)
    n_mol = len(seg) - 1
    total = int(seg[-1])
    # molecule boundaries closest to equal atom shares
    targets = [round(total * r / world) for r in range(world + 1)]
    bounds = [int(np.searchsorted(seg, t, side="left")) for t in targets]
    bounds[0], bounds[-1] = 0, n_mol
    for r in range(1, world):
        bounds[r] = max(bounds[r], bounds[r - 1])
    m0, m1 = bounds[rank], bounds[rank + 1]
    a0, a1 = int(seg[m0]), int(seg[m1])
    local = (seg[m0:m1 + 1] - a0).astype(np.int32)
    return m0, m1, a0, a1, local


# ------------------------------------------------------------------ rows
@dataclass
class RowPlan:
    """Contiguous query-row slabs, padded to equal size for the collectives."""
    N: int
    world: int

    @property
    def per(self) -> int:
        return (self.N + self.world - 1) // self.world

    def rows(self, rank: int):
        a0 = min(self.N, rank * self.per)
        return a0, min(self.N, a0 + self.per)


def _is_nccl() -> bool:
    return dist.get_backend() == "nccl"


def all_gather_rows(x_loc: torch.Tensor, plan: RowPlan, group=None) -> torch.Tensor:
    """[n_loc, ...] per rank -> [N, ...] in rank order (slabs padded to plan.per)."""
    per = plan.per
    pad = torch.zeros((per,) + tuple(x_loc.shape[1:]), dtype=x_loc.dtype, device=x_loc.device)
    pad[: x_loc.shape[0]] = x_loc
    if _is_nccl():
        out = torch.empty((per * plan.world,) + tuple(x_loc.shape[1:]), dtype=x_loc.dtype, device=x_loc.device)
        dist.all_gather_into_tensor(out, pad, group=group)
    else:
        parts = [torch.empty_like(pad) for _ in range(plan.world)]
        dist.all_gather(parts, pad, group=group)
        out = torch.cat(parts)
    return out[: plan.N]


def reduce_scatter_rows(x_all: torch.Tensor, plan: RowPlan, rank: int, group=None) -> torch.Tensor:
    """Sum [N, ...] partials over ranks and return this rank's slab."""
    per = plan.per
    pad = torch.zeros((per * plan.world,) + tuple(x_all.shape[1:]), dtype=x_all.dtype, device=x_all.device)
    pad[: plan.N] = x_all
    if _is_nccl():
        out = torch.empty((per,) + tuple(x_all.shape[1:]), dtype=x_all.dtype, device=x_all.device)
        dist.reduce_scatter_tensor(out, pad, group=group)
    else:  # gloo has no reduce_scatter: all_reduce + slice (test harness only)
        dist.all_reduce(pad, group=group)
        out = pad[rank * per:(rank + 1) * per]
    a0, a1 = plan.rows(rank)
    return out[: a1 - a0]


class CudaBackend:
    """The product backend: every call is a libequistream_b200.so kernel."""

    def __init__(self, cfg):
        from . import api
        self.api = api
        self.cfg = cfg

    def project(self, h, W):
        return self.api.project_qk(h, W, self.cfg.L)

    def project_bwd(self, h, W, dq, dk, dv):
        return self.api.project_qk_backward(h, W, self.cfg.L, dq, dk, dv)

    def attn_fwd(self, q_loc, k, v, pos, table_loc, row0):
        idx = self.api.NeighborIndex(table_loc, None, None, self.cfg.r_cut)
        keep = self.cfg.keep_scores
        res = self.api.stream_aggregate(q_loc, k, v, pos, idx, self.cfg, row0=row0, return_scores=keep)
        out, lse, sc = res if keep else (*res, None)
        idx._scores = sc  # the forward's scores (if kept) travel with the index to the backward
        return out, lse, idx

    def attn_bwd(self, g_loc, q_loc, k, v, pos, idx, out, lse, row0):
        saved = self.api.SavedAttention(q_loc, k, v, pos, idx, out, lse, self.cfg, row0=row0,
                                        scores=getattr(idx, "_scores", None))
        return self.api.stream_aggregate_backward(g_loc, saved)


def _all_gather_start(x_loc: torch.Tensor, plan: RowPlan, group=None):
    """Asynchronous all_gather_rows: returns (work, finish) -- finish() waits and
    yields the [N, ...] tensor."""
    per = plan.per
    pad = torch.zeros((per,) + tuple(x_loc.shape[1:]), dtype=x_loc.dtype, device=x_loc.device)
    pad[: x_loc.shape[0]] = x_loc
    if _is_nccl():
        out = torch.empty((per * plan.world,) + tuple(x_loc.shape[1:]), dtype=x_loc.dtype, device=x_loc.device)
        work = dist.all_gather_into_tensor(out, pad, group=group, async_op=True)
        return lambda: (work.wait(), out[: plan.N])[1]
    parts = [torch.empty_like(pad) for _ in range(plan.world)]
    work = dist.all_gather(parts, pad, group=group, async_op=True)
    return lambda: (work.wait(), torch.cat(parts)[: plan.N])[1]


def _reduce_scatter_start(x_all: torch.Tensor, plan: RowPlan, rank: int, group=None):
    """Asynchronous reduce_scatter_rows: returns finish() -> this rank's slab."""
    per = plan.per
    pad = torch.zeros((per * plan.world,) + tuple(x_all.shape[1:]), dtype=x_all.dtype, device=x_all.device)
    pad[: plan.N] = x_all
    a0, a1 = plan.rows(rank)
    if _is_nccl():
        out = torch.empty((per,) + tuple(x_all.shape[1:]), dtype=x_all.dtype, device=x_all.device)
        work = dist.reduce_scatter_tensor(out, pad, group=group, async_op=True)
        return lambda: (work.wait(), out[: a1 - a0])[1]
    work = dist.all_reduce(pad, group=group, async_op=True)  # gloo has no reduce_scatter (test harness)
    return lambda: (work.wait(), pad[rank * per:rank * per + (a1 - a0)])[1]


def interior_span(table_loc: torch.Tensor, a0: int, a1: int):
    """The longest contiguous run [b_lo, b_hi) of local rows whose neighbours all
    lie in this rank's own slab [a0, a1): those rows can run against the local
    K/V while the all-gather is in flight (x-sorted slabs: the slab's middle)."""
    t = table_loc
    inside = ((t < 0) | ((t >= a0) & (t < a1))).all(dim=1).to(torch.int8).cpu().numpy()
    best, cur, start = (0, 0), 0, 0
    for r, f in enumerate(inside):
        if f:
            if cur == 0:
                start = r
            cur += 1
            if cur > best[1] - best[0]:
                best = (start, r + 1)
        else:
            cur = 0
    return best


class RowShardedAttention:
    """One attention layer of one large system, query rows sharded over ranks.

    forward(h_loc, W, pos, table_loc) -> out_loc
    backward(g_loc) -> (dh_loc, dW)          (dW summed over ranks)
    `table_loc` is the neighbour index of this rank's rows (global key ids),
    e.g. rows [a0, a1) of build_neighbors on the replicated positions
    (es_neighbors_build with row0 / nrows).

    overlap=True (default with world > 1): the K/V all-gather runs
    asynchronously while the slab's interior rows (every neighbour inside the
    slab, `interior_span`) attend to the local K/V; the boundary rows follow
    once the gather lands.  In the backward the boundary rows' dk/dv partials
    are reduce-scattered asynchronously while the interior rows' backward
    (local keys only) runs.
    """

    def __init__(self, N: int, backend, rank: int, world: int, group=None, overlap: bool = True):
        self.plan = RowPlan(N, world)
        self.backend = backend
        self.rank, self.world, self.group = rank, world, group
        self.a0, self.a1 = self.plan.rows(rank)
        self.overlap = (overlap and world > 1) or overlap == "force"  # "force": exercise the path at world 1
        self._span_key = None

    def _span(self, table_loc):
        key = (table_loc.data_ptr(), tuple(table_loc.shape))
        if self._span_key != key:
            self._span_val = interior_span(table_loc, self.a0, self.a1)
            self._span_key = key
        return self._span_val

    def _local_pos(self, pos):
        p = pos[self.a0:self.a1]
        return p if p.data_ptr() % 16 == 0 else p.contiguous().clone()  # es_attn_fwd: 16-byte aligned

    def forward(self, h_loc, W, pos, table_loc):
        q, k_loc, v_loc = self.backend.project(h_loc, W)
        b_lo, b_hi = self._span(table_loc) if self.overlap else (0, 0)
        if b_hi <= b_lo:  # nothing to overlap: one blocking all-gather per layer
            k = all_gather_rows(k_loc, self.plan, self.group)
            v = all_gather_rows(v_loc, self.plan, self.group)
            out, lse, idx = self.backend.attn_fwd(q, k, v, pos, table_loc, self.a0)
            self._saved = (h_loc, W, q, k, v, pos, [(0, q.shape[0], idx, False)], out, lse)
            return out
        fin_k = _all_gather_start(k_loc, self.plan, self.group)
        fin_v = _all_gather_start(v_loc, self.plan, self.group)
        # interior rows against the local keys (ids remapped into the slab) while the gather is in flight
        t_int = table_loc[b_lo:b_hi]
        t_int = torch.where(t_int >= 0, t_int - self.a0, t_int).contiguous()
        pos_loc = self._local_pos(pos)
        o_i, l_i, idx_i = self.backend.attn_fwd(q[b_lo:b_hi].contiguous(), k_loc, v_loc, pos_loc, t_int, b_lo)
        k, v = fin_k(), fin_v()
        outs, lses, parts = [], [], []
        for r0, r1, interior in ((0, b_lo, False), (b_lo, b_hi, True), (b_hi, q.shape[0], False)):
            if r1 <= r0:
                continue
            if interior:
                outs.append(o_i); lses.append(l_i); parts.append((r0, r1, idx_i, True))
                continue
            o_b, l_b, idx_b = self.backend.attn_fwd(q[r0:r1].contiguous(), k, v, pos, table_loc[r0:r1].contiguous(),
                                                    self.a0 + r0)
            outs.append(o_b); lses.append(l_b); parts.append((r0, r1, idx_b, False))
        out, lse = torch.cat(outs), torch.cat(lses)
        self._saved = (h_loc, W, q, k, v, pos, parts, out, lse)
        return out

    def backward(self, g_loc):
        h_loc, W, q, k, v, pos, parts, out, lse = self._saved
        acc = torch.float32 if k.dtype in (torch.bfloat16, torch.float16) else k.dtype  # sum in >= fp32
        dq = torch.empty_like(q)
        dk_all = dv_all = None
        for r0, r1, idx, interior in parts:  # boundary rows first: their partials go out asynchronously
            if interior:
                continue
            dq_b, dk_b, dv_b = self.backend.attn_bwd(g_loc[r0:r1].contiguous(), q[r0:r1].contiguous(), k, v, pos, idx,
                                                     out[r0:r1].contiguous(), lse[r0:r1].contiguous(), self.a0 + r0)
            dq[r0:r1] = dq_b
            dk_all = dk_b.to(acc) if dk_all is None else dk_all + dk_b.to(acc)
            dv_all = dv_b.to(acc) if dv_all is None else dv_all + dv_b.to(acc)
        if dk_all is None:  # every row interior: the other ranks still expect this rank's (zero) partials
            dk_all = torch.zeros(k.shape, dtype=acc, device=k.device)
            dv_all = torch.zeros(v.shape, dtype=acc, device=v.device)
        fin_dk = _reduce_scatter_start(dk_all, self.plan, self.rank, self.group)
        fin_dv = _reduce_scatter_start(dv_all, self.plan, self.rank, self.group)
        dk_int = dv_int = None
        for r0, r1, idx, interior in parts:  # interior rows (local keys) overlap the reduce-scatter
            if not interior:
                continue
            n_loc = self.a1 - self.a0
            dq_i, dk_int, dv_int = self.backend.attn_bwd(g_loc[r0:r1].contiguous(), q[r0:r1].contiguous(),
                                                         k[self.a0:self.a1].contiguous(),
                                                         v[self.a0:self.a1].contiguous(), self._local_pos(pos), idx,
                                                         out[r0:r1].contiguous(), lse[r0:r1].contiguous(), r0)
            assert dk_int.shape[0] == n_loc
            dq[r0:r1] = dq_i
        dk, dv = fin_dk(), fin_dv()
        if dk_int is not None:
            dk = dk + dk_int.to(acc)
            dv = dv + dv_int.to(acc)
        dk, dv = dk.to(k.dtype), dv.to(v.dtype)
        dh, dW = self.backend.project_bwd(h_loc, W, dq, dk.contiguous(), dv.contiguous())
        if dW is not None:
            dist.all_reduce(dW, group=self.group)
        return dh, dW


# ------------------------------------------------------------------ halo exchange
def _all_to_all_rows(send: torch.Tensor, send_counts, recv_counts, group=None) -> torch.Tensor:
    """Variable-size all-to-all of row blocks (rows for rank r' contiguous in
    `send`).  NCCL: all_to_all_single; gloo (test harness): all_gather of
    padded blocks."""
    tail = tuple(send.shape[1:])
    if _is_nccl():
        out = torch.empty((int(sum(recv_counts)),) + tail, dtype=send.dtype, device=send.device)
        dist.all_to_all_single(out, send.contiguous(), output_split_sizes=list(map(int, recv_counts)),
                               input_split_sizes=list(map(int, send_counts)), group=group)
        return out
    world = len(send_counts)
    rank = dist.get_rank(group)
    cap = max(1, max(int(max(send_counts)), 0))
    caps = torch.tensor([cap], dtype=torch.int64)
    allc = [torch.zeros_like(caps) for _ in range(world)]
    dist.all_gather(allc, caps, group=group)
    cap = int(max(c.item() for c in allc))
    blocks = torch.zeros((world, cap) + tail, dtype=send.dtype)
    off = 0
    for r in range(world):
        n = int(send_counts[r])
        blocks[r, :n] = send[off:off + n]
        off += n
    parts = [torch.empty_like(blocks) for _ in range(world)]
    dist.all_gather(parts, blocks, group=group)
    return torch.cat([parts[r][rank, :int(recv_counts[r])] for r in range(world)])


class HaloPlan:
    """Which K/V rows of other ranks' slabs this rank's query rows touch.

    Built once per neighbour list: the rank's key set is its own slab plus the
    halo (every neighbour id outside the slab), in a compact index space --
    own rows first (so row0 = 0), then halo atoms grouped by owner.  The
    forward then exchanges only halo rows (all-to-all) instead of all-gathering
    every atom: at 100k atoms on 8 GPUs a 14 A slab plus 2 x 6 A of halo
    instead of the whole box.  The backward sends
    the halo rows' dk / dv partials back to their owners and sums them there.
    """

    def __init__(self, table_loc: torch.Tensor, plan: RowPlan, rank: int, world: int, group=None):
        self.plan, self.rank, self.world, self.group = plan, rank, world, group
        a0, a1 = plan.rows(rank)
        self.a0, self.n_loc = a0, a1 - a0
        ids = torch.unique(table_loc[table_loc >= 0].long())
        halo = ids[(ids < a0) | (ids >= a1)]
        owner = torch.div(halo, plan.per, rounding_mode="floor")
        self.halo = halo  # ascending = grouped by owner
        # collectives run on the table's device (NCCL) or the CPU (gloo test harness)
        cdev = table_loc.device if _is_nccl() else torch.device("cpu")
        req = torch.bincount(owner.to(cdev), minlength=world)[:world].to(torch.int64)
        counts = [torch.zeros_like(req) for _ in range(world)]
        dist.all_gather(counts, req, group=group)  # counts[src][dst]: rows src needs from dst
        self.recv_counts = [int(counts[rank][r]) for r in range(world)]  # halo rows I receive, per owner
        self.send_counts = [int(counts[r][rank]) for r in range(world)]  # my rows each requester needs
        asked = _all_to_all_rows(halo.to(cdev).view(-1, 1), self.recv_counts, self.send_counts, group)
        self.send_rows = (asked.view(-1).to(table_loc.device) - a0).long()  # local rows to send, by requester
        gmap = torch.full((plan.N,), -1, dtype=torch.int64, device=table_loc.device)
        gmap[a0:a1] = torch.arange(self.n_loc, device=table_loc.device)
        gmap[halo.to(table_loc.device)] = self.n_loc + torch.arange(len(halo), device=table_loc.device)
        t = table_loc.long()
        self.table = torch.where(t >= 0, gmap[t.clamp(min=0)], t).to(table_loc.dtype)
        self.keys = torch.cat([torch.arange(a0, a1, device=table_loc.device), halo.to(table_loc.device)])

    @property
    def n_keys(self) -> int:
        return self.n_loc + len(self.halo)

    def gather(self, x_loc: torch.Tensor) -> torch.Tensor:
        """Own rows + the halo rows from their owners -> [n_keys, ...]."""
        halo_rows = _all_to_all_rows(x_loc[self.send_rows], self.send_counts, self.recv_counts, self.group)
        return torch.cat([x_loc, halo_rows.to(x_loc.device)])

    def scatter_add(self, x_keys: torch.Tensor) -> torch.Tensor:
        """Partials over [n_keys, ...] -> summed partials of this rank's rows."""
        back = _all_to_all_rows(x_keys[self.n_loc:], self.recv_counts, self.send_counts, self.group)
        own = x_keys[: self.n_loc].clone()
        own.index_add_(0, self.send_rows, back.to(own.device))
        return own


class HaloShardedAttention(RowShardedAttention):
    """RowShardedAttention with a halo exchange instead of the K/V all-gather:
    per layer each rank receives only the K/V rows its neighbour lists touch
    and returns only their dk / dv partials."""

    def forward(self, h_loc, W, pos, table_loc):
        self.halo = HaloPlan(table_loc, self.plan, self.rank, self.world, self.group)
        q, k_loc, v_loc = self.backend.project(h_loc, W)
        k = self.halo.gather(k_loc)
        v = self.halo.gather(v_loc)
        pos_c = pos[self.halo.keys.to(pos.device)]
        out, lse, idx = self.backend.attn_fwd(q, k, v, pos_c, self.halo.table, 0)
        self._saved = (h_loc, W, q, k, v, pos_c, idx, out, lse)
        return out

    def backward(self, g_loc):
        h_loc, W, q, k, v, pos_c, idx, out, lse = self._saved
        dq, dk_c, dv_c = self.backend.attn_bwd(g_loc, q, k, v, pos_c, idx, out, lse, 0)
        acc = torch.float32 if dk_c.dtype in (torch.bfloat16, torch.float16) else dk_c.dtype
        dk = self.halo.scatter_add(dk_c.to(acc)).to(dk_c.dtype)
        dv = self.halo.scatter_add(dv_c.to(acc)).to(dv_c.dtype)
        dh, dW = self.backend.project_bwd(h_loc, W, dq, dk.contiguous(), dv.contiguous())
        if dW is not None:
            dist.all_reduce(dW, group=self.group)
        return dh, dW
