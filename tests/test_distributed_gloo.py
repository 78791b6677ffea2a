"""Multi-process (world_size 2, gloo, CPU) checks of the sharding logic in
paper_2601_16622_b200.distributed: molecule-batch partition and query-row
sharding with the K/V all-gather and dk/dv reduce-scatter, with the CPU
oracle standing in for the per-rank GPU compute (test-only backend)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po
from paper_2601_16622_b200 import distributed as D
from paper_2601_16622_b200 import systems as S

L, C, H, K = 1, 8, 2, 32


class OracleBackend:
    """Per-rank compute on the CPU oracle (row0 emulated by padding)."""

    def __init__(self, N, box=None):
        self.N = N
        self.P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_DENSE, box=box)

    def project(self, h, W):
        return tuple(torch.from_numpy(x) for x in po.project(h.numpy(), W.numpy(), L))

    def project_bwd(self, h, W, dq, dk, dv):
        dh, dW = po.project_bwd(h.numpy(), W.numpy(), L, dq.numpy(), dk.numpy(), dv.numpy())
        return torch.from_numpy(dh), torch.from_numpy(dW)

    def _full(self, x_loc, row0, n=None):
        full = np.zeros((n or self.N,) + tuple(x_loc.shape[1:]), dtype=np.float64)
        full[row0:row0 + x_loc.shape[0]] = x_loc
        return full

    def attn_fwd(self, q_loc, k, v, pos, table_loc, row0):
        nk = k.shape[0]  # all atoms (all-gather), own slab (overlapped interior rows) or slab + halo
        nbr = -np.ones((nk, table_loc.shape[1]), np.int32)
        nbr[row0:row0 + len(table_loc)] = table_loc.numpy()
        out, lse = po.attn_fwd(self.P, self._full(q_loc.numpy(), row0, nk), k.numpy(), v.numpy(), pos.numpy(), nbr)
        n = len(table_loc)
        ctx = (nbr, out, lse)  # travels as the "index" of this call to its backward
        return torch.from_numpy(out[row0:row0 + n]), torch.from_numpy(lse[row0:row0 + n]), ctx

    def attn_bwd(self, g_loc, q_loc, k, v, pos, idx, out, lse, row0):
        nbr, out_f, lse_f = idx
        nk = k.shape[0]
        dq, dk, dv = po.attn_bwd(self.P, self._full(q_loc.numpy(), row0, nk), k.numpy(), v.numpy(), pos.numpy(), nbr,
                                 out_f, lse_f, self._full(g_loc.numpy(), row0, nk))
        n = q_loc.shape[0]
        return torch.from_numpy(dq[row0:row0 + n]), torch.from_numpy(dk), torch.from_numpy(dv)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _system():
    b = S.periodic_box(90, 3, 3.8, 4)  # 108 sites, box 11.4 A (minimum image, brute force)
    h = S.random_features(len(b.pos), L, C, 4)
    W = S.random_weights(L, C, 4)
    g = np.random.default_rng(5).standard_normal((len(b.pos), (L + 1) ** 2, C))
    return b, h, W, g


def _row_worker(rank, world, port, outdir, halo=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, h, W, g = _system()
    N = len(b.pos)
    nbr, _, _ = po.build_neighbors(b.pos, K, 6.0, box=b.box)
    cls = D.HaloShardedAttention if halo else D.RowShardedAttention
    layer = cls(N, OracleBackend(N, b.box), rank, world)
    a0, a1 = layer.a0, layer.a1
    out = layer.forward(torch.from_numpy(h[a0:a1].copy()), torch.from_numpy(W), torch.from_numpy(b.pos),
                        torch.from_numpy(nbr[a0:a1].copy()))
    dh, dW = layer.backward(torch.from_numpy(g[a0:a1].copy()))
    out_all = D.all_gather_rows(out, layer.plan)
    dh_all = D.all_gather_rows(dh, layer.plan)
    if rank == 0:
        extra = {"n_keys": layer.halo.n_keys} if halo else {}
        np.savez(os.path.join(outdir, "row.npz"), out=out_all.numpy(), dh=dh_all.numpy(), dW=dW.numpy(), **extra)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,halo", [(2, False), (2, True), (3, True)])
def test_row_sharding_gloo_matches_unsharded(tmp_path, oracle, world, halo):
    mp.spawn(_row_worker, args=(world, _free_port(), str(tmp_path), halo), nprocs=world, join=True)
    got = np.load(tmp_path / "row.npz")
    b, h, W, g = _system()
    nbr, _, _ = po.build_neighbors(b.pos, K, 6.0, box=b.box)
    P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_DENSE, box=b.box)
    q, k, v = po.project(h, W, L)
    out, lse = po.attn_fwd(P, q, k, v, b.pos, nbr)
    dq, dk, dv = po.attn_bwd(P, q, k, v, b.pos, nbr, out, lse, g)
    dh, dW = po.project_bwd(h, W, L, dq, dk, dv)
    np.testing.assert_allclose(got["out"], out, atol=1e-12 * np.abs(out).max())
    np.testing.assert_allclose(got["dh"], dh, atol=1e-12 * np.abs(dh).max())
    np.testing.assert_allclose(got["dW"], dW, atol=1e-12 * np.abs(dW).max())


def _overlap_worker(rank, world, port, outdir):
    """x-sorted open FCC system: each slab has interior rows (every neighbour in
    the slab) that attend to the local K/V while the all-gather is in flight."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos = S.gen_fcc_system(400, 3.8, 7)  # site order: x-major -> slabs are x-slabs
    N = len(pos)
    h = S.random_features(N, L, C, 8)
    W = S.random_weights(L, C, 8)
    g = np.random.default_rng(9).standard_normal((N, (L + 1) ** 2, C))
    nbr, _, _ = po.build_neighbors(pos, K, 6.0)
    layer = D.RowShardedAttention(N, OracleBackend(N), rank, world)
    a0, a1 = layer.a0, layer.a1
    tl = torch.from_numpy(nbr[a0:a1].copy())
    span = D.interior_span(tl, a0, a1)
    out = layer.forward(torch.from_numpy(h[a0:a1].copy()), torch.from_numpy(W), torch.from_numpy(pos), tl)
    dh, dW = layer.backward(torch.from_numpy(g[a0:a1].copy()))
    out_all = D.all_gather_rows(out, layer.plan)
    dh_all = D.all_gather_rows(dh, layer.plan)
    sp = torch.tensor([span[0], span[1]], dtype=torch.int64)
    spans = [torch.zeros_like(sp) for _ in range(world)]
    dist.all_gather(spans, sp)
    if rank == 0:
        np.savez(os.path.join(outdir, "ovl.npz"), out=out_all.numpy(), dh=dh_all.numpy(), dW=dW.numpy(),
                 spans=np.stack([x.numpy() for x in spans]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharding_overlapped_gather_gloo(tmp_path, oracle, world):
    """RowShardedAttention(overlap=True): interior rows run before the K/V
    all-gather lands, boundary partials are reduce-scattered while the interior
    backward runs -- identical to the unsharded layer."""
    mp.spawn(_overlap_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "ovl.npz")
    # the end slabs have rows to overlap (a thin middle slab of world 3 has none: every row sees both faces)
    assert got["spans"][0, 1] > got["spans"][0, 0] and got["spans"][-1, 1] > got["spans"][-1, 0]
    pos = S.gen_fcc_system(400, 3.8, 7)
    h = S.random_features(len(pos), L, C, 8)
    W = S.random_weights(L, C, 8)
    g = np.random.default_rng(9).standard_normal((len(pos), (L + 1) ** 2, C))
    nbr, _, _ = po.build_neighbors(pos, K, 6.0)
    P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_DENSE)
    q, k, v = po.project(h, W, L)
    out, lse = po.attn_fwd(P, q, k, v, pos, nbr)
    dq, dk, dv = po.attn_bwd(P, q, k, v, pos, nbr, out, lse, g)
    dh, dW = po.project_bwd(h, W, L, dq, dk, dv)
    np.testing.assert_allclose(got["out"], out, atol=1e-12 * np.abs(out).max())
    np.testing.assert_allclose(got["dh"], dh, atol=1e-12 * np.abs(dh).max())
    np.testing.assert_allclose(got["dW"], dW, atol=1e-12 * np.abs(dW).max())


def _mol_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = S.molecule_batch(9, 10, 30, seed=2)
    m0, m1, a0, a1, seg = D.shard_molecules(batch.seg_ptr, world, rank)
    pos = batch.pos[a0:a1]
    nbr, _, _ = po.build_neighbors(pos, K, 6.0, seg_ptr=seg)
    h = S.random_features(batch.n_atoms, L, C, 3)[a0:a1]
    q, k, v = po.project(h, S.random_weights(L, C, 3), L)
    out, _ = po.attn_fwd(po.AttnProblem(L=L, H=H), q, k, v, pos, nbr)
    t = torch.zeros(2, dtype=torch.int64)
    t[0], t[1] = a0, a1
    spans = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(spans, t)  # bookkeeping only: molecules need no data-path collective
    np.savez(os.path.join(outdir, f"mol{rank}.npz"), out=out, a0=a0, a1=a1,
             spans=np.stack([s.numpy() for s in spans]))
    dist.barrier()
    dist.destroy_process_group()


def test_molecule_sharding_gloo(tmp_path, oracle):
    world = 2
    mp.spawn(_mol_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    batch = S.molecule_batch(9, 10, 30, seed=2)
    nbr, _, _ = po.build_neighbors(batch.pos, K, 6.0, seg_ptr=batch.seg_ptr)
    q, k, v = po.project(S.random_features(batch.n_atoms, L, C, 3), S.random_weights(L, C, 3), L)
    ref, _ = po.attn_fwd(po.AttnProblem(L=L, H=H), q, k, v, batch.pos, nbr)
    covered = 0
    for r in range(world):
        d = np.load(tmp_path / f"mol{r}.npz")
        a0, a1 = int(d["a0"]), int(d["a1"])
        np.testing.assert_allclose(d["out"], ref[a0:a1], atol=1e-12 * np.abs(ref).max())
        covered += a1 - a0
        spans = d["spans"]
        assert spans[0][0] == 0 and spans[-1][1] == batch.n_atoms and spans[0][1] == spans[1][0]
    assert covered == batch.n_atoms


def test_shard_molecules_balance():
    seg = np.concatenate([[0], np.cumsum(np.random.default_rng(0).integers(40, 61, 4096))]).astype(np.int32)
    sizes = []
    for r in range(8):
        m0, m1, a0, a1, local = D.shard_molecules(seg, 8, r)
        assert local[0] == 0 and local[-1] == a1 - a0
        sizes.append(a1 - a0)
    assert sum(sizes) == seg[-1] and max(sizes) - min(sizes) <= 120


def _halo_size_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos = S.gen_fcc_system(4000, 3.8, 7)
    pos = pos[np.argsort(pos[:, 0], kind="stable")]  # slabs along x: spatially contiguous row shards
    nbr, _, _ = po.build_neighbors(pos, 64, 6.0)
    plan = D.RowPlan(len(pos), world)
    a0, a1 = plan.rows(rank)
    hp = D.HaloPlan(torch.from_numpy(nbr[a0:a1].copy()), plan, rank, world)
    x = torch.arange(a1 - a0, dtype=torch.float64).view(-1, 1) + a0  # row value = its global id
    keys_val = hp.gather(x)
    ok = bool(torch.equal(keys_val.view(-1).long(), hp.keys.long()))
    summed = hp.scatter_add(torch.ones(hp.n_keys, 1, dtype=torch.float64))
    np.savez(os.path.join(outdir, f"halo{rank}.npz"), n_keys=hp.n_keys, n_loc=a1 - a0, ok=ok,
             summed=summed.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_halo_plan_exchanges_only_the_halo(tmp_path):
    """4 slabs of a 4000-atom system: each rank receives a halo far smaller
    than the system, gather returns every key's row, and scatter_add counts
    each row once for its owner plus once per rank that holds it as halo."""
    world = 4
    mp.spawn(_halo_size_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    total_halo_copies = 0
    for r in range(world):
        d = np.load(tmp_path / f"halo{r}.npz")
        assert bool(d["ok"])
        assert int(d["n_keys"]) < 0.75 * 4000
        total_halo_copies += int(d["n_keys"]) - int(d["n_loc"])
    summed = np.concatenate([np.load(tmp_path / f"halo{r}.npz")["summed"] for r in range(world)])
    assert summed.min() >= 1 and summed.sum() == 4000 + total_halo_copies
