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


class RowShardedAttention:
    """One attention layer of one large system, query rows sharded over ranks.

    forward(h_loc, W, pos, table_loc) -> out_loc
    backward(g_loc) -> (dh_loc, dW)          (dW summed over ranks)
    `table_loc` is the neighbour index of this rank's rows (global key ids),
    e.g. rows [a0, a1) of build_neighbors on the replicated positions.
    """

    def __init__(self, N: int, backend, rank: int, world: int, group=None):
        self.plan = RowPlan(N, world)
        self.backend = backend
        self.rank, self.world, self.group = rank, world, group
        self.a0, self.a1 = self.plan.rows(rank)

    def forward(self, h_loc, W, pos, table_loc):
        q, k_loc, v_loc = self.backend.project(h_loc, W)
        k = all_gather_rows(k_loc, self.plan, self.group)  # one K/V all-gather per layer
        v = all_gather_rows(v_loc, self.plan, self.group)
        out, lse, idx = self.backend.attn_fwd(q, k, v, pos, table_loc, self.a0)
        self._saved = (h_loc, W, q, k, v, pos, idx, out, lse)
        return out

    def backward(self, g_loc):
        h_loc, W, q, k, v, pos, idx, out, lse = self._saved
        dq, dk_all, dv_all = self.backend.attn_bwd(g_loc, q, k, v, pos, idx, out, lse, self.a0)
        acc = torch.float32 if dk_all.dtype in (torch.bfloat16, torch.float16) else dk_all.dtype  # sum in >= fp32
        dk = reduce_scatter_rows(dk_all.to(acc), self.plan, self.rank, self.group).to(dk_all.dtype)
        dv = reduce_scatter_rows(dv_all.to(acc), self.plan, self.rank, self.group).to(dv_all.dtype)
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
