"""The E2Former-V2 attention block as one autograd op:
projections (Eq. 6 + W_H) -> fused streaming attention with per-pair EAAS
-> output, with the recompute backward of both.  Every launch is a kernel
of libequistream_b200.so."""
from __future__ import annotations

import torch

from .api import (AttentionConfig, NeighborIndex, SavedAttention, project_qk, project_qk_backward,
                  stream_aggregate, stream_aggregate_backward)


class _AttnFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, h, W, pos, idx: NeighborIndex, cfg: AttentionConfig):
        q, k, v = project_qk(h.contiguous(), W.contiguous(), cfg.L)
        res = stream_aggregate(q, k, v, pos, idx, cfg, return_scores=cfg.keep_scores)
        out, lse, scores = res if cfg.keep_scores else (*res, None)
        ctx.save_for_backward(h, W, q, k, v, out, lse, pos)
        ctx.scores = scores
        ctx.idx, ctx.cfg = idx, cfg
        return out

    @staticmethod
    def backward(ctx, grad_out):
        h, W, q, k, v, out, lse, pos = ctx.saved_tensors
        saved = SavedAttention(q, k, v, pos, ctx.idx, out, lse, ctx.cfg, scores=ctx.scores)
        want_pos = ctx.needs_input_grad[2]  # positions require grad: forces
        grads = stream_aggregate_backward(grad_out.contiguous().to(q.dtype), saved, pos_grad=want_pos)
        dq, dk, dv = grads[:3]
        dh, dW = project_qk_backward(h, W, ctx.cfg.L, dq, dk, dv, want_dW=ctx.needs_input_grad[1])
        dpos = grads[3].to(pos.dtype) if want_pos else None
        return dh, (dW.to(W.dtype) if dW is not None else None), dpos, None, None


def attention_layer(h: torch.Tensor, W: torch.Tensor, pos: torch.Tensor, idx: NeighborIndex,
                    cfg: AttentionConfig) -> torch.Tensor:
    return _AttnFn.apply(h, W, pos, idx, cfg)


class EquivariantAttention(torch.nn.Module):
    """Per-degree W = [W_Q1 | W_Q2 | W_K1 | W_K2 | W_H] ~ N(0, 1/C)."""

    def __init__(self, L: int, channels: int, heads: int, r_cut: float = 6.0, value_mode: str = "eaas",
                 dtype=torch.float32, device="cuda"):
        super().__init__()
        self.cfg = AttentionConfig(heads=heads, L=L, r_cut=r_cut, value_mode=value_mode)
        w = torch.randn(L + 1, channels, 5 * channels, device=device) / channels ** 0.5
        self.W = torch.nn.Parameter(w.to(dtype))

    def forward(self, h, pos, idx: NeighborIndex, box=None):
        cfg = self.cfg if box is None else AttentionConfig(**{**self.cfg.__dict__, "box": tuple(box)})
        return attention_layer(h, self.W, pos, idx, cfg)
