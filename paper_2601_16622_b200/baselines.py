"""Comparison baselines of the paper's Fig. 1-3 on the GPU,
written in plain PyTorch on purpose: they are what the fused kernel is
measured against, not part of the product path.

* ``edge_materialising_attention`` -- the edge-centric formulation
  (Eq. 4; SPEC edge_centric_message SPEC.md:342-350):
  every neighbour pair gets its own tensors (gathered q/k/v rows, scores,
  the dense Clebsch-Gordan product of v_j with the solid harmonics of r_ij)
  before the softmax-weighted sum.  Memory O(E * M * C) per processed row
  chunk; the dense CG contraction costs M^3 = 729 MACs per pair-channel at
  L = 2 (615 non-trivial in the paper's count) instead of EAAS's 107.
* ``masked_dense_attention`` -- global scaled-dot-product attention over all
  N x N pairs with the neighbour mask, plain values (no
  geometry); O(N^2) scores.

Both follow the library's conventions (irreps layout [N][M][C], head h owns
q/k channels [h*2C/H, (h+1)*2C/H) and value channels [h*C/H, (h+1)*C/H) of
every (l, m) row, tau = 1/sqrt(d_k), phi = cosine cutoff), so their outputs
equal ``stream_aggregate``'s up to rounding (tests/test_gpu_baselines.py).
"""
from __future__ import annotations

import math

import torch

from . import _lib

# solid harmonic constants of the library (attention_common.cuh solid2_grad)
_C0, _C1, _C2, _C20 = 0.28209479177387814, 0.4886025119029199, 1.0925484305920792, 0.6307831305050401


def coupling_tensor(L: int = 2, device="cuda", dtype=torch.float32) -> torch.Tensor:
    """G[o, i, f] = cg_real(l_i, l_f, l_o)[m_o](m_i, m_f) over the path set
    (every triangle-valid (l_i, l_f, l_o) with all degrees <= L, weight 1)."""
    M = (L + 1) ** 2
    deg = [int(math.isqrt(x)) for x in range(M)]
    lib = _lib.lib()
    G = torch.zeros(M, M, M, dtype=torch.float64)
    for o in range(M):
        for i in range(M):
            for f in range(M):
                lo, li, lf = deg[o], deg[i], deg[f]
                G[o, i, f] = lib.es_cg_real(li, i - li * li - li, lf, f - lf * lf - lf, lo, o - lo * lo - lo)
    return G.to(device=device, dtype=dtype)


def solid_harmonics_l2(r: torch.Tensor) -> torch.Tensor:
    """Y^f(r), f = 0..8 (rows l*l + m + l), for r [..., 3]."""
    x, y, z = r[..., 0], r[..., 1], r[..., 2]
    return torch.stack([torch.full_like(x, _C0), _C1 * y, _C1 * z, -_C1 * x, _C2 * x * y, _C2 * y * z,
                        _C20 * (z * z - 0.5 * (x * x + y * y)), -_C2 * x * z, 0.5 * _C2 * (x * x - y * y)], -1)


def _pair_vectors(pos, nbr, rows, box):
    j = nbr[rows].long()
    valid = j >= 0
    jj = torch.where(valid, j, torch.zeros_like(j))
    d = pos[jj] - pos[rows].unsqueeze(1)
    if box is not None:
        b = torch.tensor(box, dtype=d.dtype, device=d.device)
        d = d - b * torch.round(d / b)
    return jj, valid, d


def edge_materialising_attention(q, k, v, pos, nbr, heads: int, L: int = 2, r_cut: float = 6.0, box=None,
                                 chunk: int = 8192, value: str = "eaas"):
    """Forward of the attention with explicit per-edge tensors (row chunks of
    `chunk` query atoms at a time).  Returns (out [N][M][C] in v's dtype,
    peak bytes of the per-edge tensors of one chunk)."""
    N, M, C = v.shape
    H = heads
    dqh = q.shape[2] // H
    ch = C // H
    tau = 1.0 / math.sqrt(M * dqh)
    G = coupling_tensor(L, q.device) if value == "eaas" else None
    outs = []  # chunk outputs concatenated (autograd-friendly: the backward baseline differentiates this)
    peak = 0
    for a in range(0, N, chunk):
        rows = torch.arange(a, min(N, a + chunk), device=q.device)
        jj, valid, d = _pair_vectors(pos, nbr, rows, box)
        n, K = jj.shape
        qi = q[rows].float().view(n, 1, M, H, dqh)
        kj = k[jj].float().view(n, K, M, H, dqh)                     # per-edge keys
        s = tau * torch.einsum("nomhd,nkmhd->nkh", qi, kj)            # [n, K, H]
        s = s.masked_fill(~valid.unsqueeze(-1), float("-inf"))
        p = torch.softmax(s, dim=1).nan_to_num(0.0)                    # zero-neighbour rows -> 0
        rn = d.norm(dim=-1).float()
        phi = torch.where(rn < r_cut, 0.5 * (torch.cos(math.pi * rn / r_cut) + 1.0), torch.zeros_like(rn))
        vj = v[jj].float()                                              # [n, K, M, C] per-edge values
        if G is not None:
            Y = solid_harmonics_l2(d.float())                           # [n, K, 9]
            x = torch.einsum("oif,nkf,nkic->nkoc", G, Y, vj)            # dense CG product per edge
        else:
            x = vj
        x = x * phi[..., None, None]
        w = p.repeat_interleave(ch, dim=2)                              # [n, K, C] head weights per channel
        outs.append(torch.einsum("nkc,nkoc->noc", w, x).to(v.dtype))
        peak = max(peak, sum(t.numel() * t.element_size() for t in (kj, s, vj, x)))
    return torch.cat(outs), peak


def baseline_backward(fn, q, k, v, grad_out):
    """The backward of a baseline by autograd through its materialised graph
    (every per-edge tensor of the forward is kept for it): (dq, dk, dv)."""
    qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))
    out = fn(qq, kk, vv)
    out.backward(grad_out)
    return qq.grad, kk.grad, vv.grad


def masked_dense_attention(q, k, v, nbr, heads: int):
    """Dense N x N scaled-dot-product attention restricted to the neighbour
    lists by a boolean mask (plain values, no geometry), through
    torch.nn.functional.scaled_dot_product_attention."""
    N, M, C = v.shape
    H = heads
    dqh = q.shape[2] // H
    mask = torch.zeros(N, N, dtype=torch.bool, device=q.device)
    rows = torch.arange(N, device=q.device).unsqueeze(1).expand_as(nbr)
    ok = nbr >= 0
    mask[rows[ok], nbr[ok].long()] = True
    qh = q.view(N, M, H, dqh).permute(2, 0, 1, 3).reshape(H, N, M * dqh)
    kh = k.view(N, M, H, dqh).permute(2, 0, 1, 3).reshape(H, N, M * dqh)
    vh = v.view(N, M, H, C // H).permute(2, 0, 1, 3).reshape(H, N, M * (C // H))
    o = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, attn_mask=mask)
    o = o.nan_to_num(0.0).view(H, N, M, C // H).permute(1, 2, 0, 3).reshape(N, M, C)
    return o
