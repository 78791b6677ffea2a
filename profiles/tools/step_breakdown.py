"""Per-phase CUDA-event breakdown of one bench step (configs[1]) -- finds
gaps between the library calls (host overhead, allocator) that the per-kernel
launch list does not show.  python profiles/tools/step_breakdown.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2601_16622_b200 as es  # noqa: E402
from paper_2601_16622_b200 import systems  # noqa: E402
from paper_2601_16622_b200.api import AttentionConfig, SavedAttention  # noqa: E402

dev = torch.device("cuda", 0)
b = systems.molecule_batch(4096, 40, 60, systems.default_seed(0))
N = b.n_atoms
rng = np.random.default_rng(0)
pos = torch.tensor(b.pos, device=dev)
seg = torch.tensor(b.seg_ptr, device=dev)
h = torch.tensor(rng.standard_normal((N, 9, 128)), device=dev).bfloat16()
W = torch.tensor(rng.standard_normal((3, 128, 640)) / np.sqrt(128), device=dev).bfloat16()
g = torch.tensor(rng.standard_normal((N, 9, 128)), device=dev).bfloat16()
cfg = AttentionConfig(heads=8, L=2, r_cut=6.0, value_mode="eaas")


def step(ev):
    ev[0].record()
    idx = es.build_neighbors(pos, 64, 6.0, seg, with_distances=False)
    ev[1].record()
    idx.transpose()
    ev[2].record()
    q, k, v = es.project_qk(h, W, 2)
    ev[3].record()
    out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
    ev[4].record()
    dq, dk, dv = es.stream_aggregate_backward(g, SavedAttention(q, k, v, pos, idx, out, lse, cfg))
    ev[5].record()
    dh, dW = es.project_qk_backward(h, W, 2, dq, dk, dv)
    ev[6].record()


names = ["neighbors", "transpose", "proj_fwd", "attn_fwd", "attn_bwd", "proj_bwd"]
for it in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    step(ev)
    torch.cuda.synchronize()
    if it >= 2:
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(6)]
        print(" ".join(f"{n}={x:.3f}" for n, x in zip(names, t)), f"total={ev[0].elapsed_time(ev[6]):.3f} ms")
