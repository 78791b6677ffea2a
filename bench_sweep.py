#!/usr/bin/env python
"""Latency / TFLOPS vs N sweep over the BASELINE.json configurations
(secondary to bench.py, whose single line is the driver's contract).

    python bench_sweep.py [--configs 1,3,4,5] [--steps 5] [--warmup 3] [--dtype bf16]

One JSON line per (config, N): fwd+bwd step latency (neighbours +
projections + attention fwd + recompute bwd + projection bwd), algorithmic
TFLOP/s, peak device memory, and -- for the small configs -- the CPU oracle
port timed on the same inputs.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def flops(n_atoms, n_pairs, L, C, H):
    M = (L + 1) ** 2
    dk, ch = 2 * M * C // H, C // H
    proj = 2 * n_atoms * M * C * 5 * C
    return 3 * proj + n_pairs * H * (2 * dk + 2 * ch * M * M) + n_pairs * H * (6 * dk + 4 * ch * M * M)


def run(system, L, C, H, K, dtype, steps, warmup, cpu=False):
    import torch

    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200.api import AttentionConfig, SavedAttention

    dev = torch.device("cuda")
    N = system.n_atoms
    M = (L + 1) ** 2
    rng = np.random.default_rng(0)
    pos = torch.tensor(system.pos, device=dev)
    seg = None if system.seg_ptr is None else torch.tensor(system.seg_ptr, device=dev)
    box = None if system.box is None else tuple(system.box)
    h = torch.tensor(rng.standard_normal((N, M, C)), device=dev).to(dtype)
    W = torch.tensor(rng.standard_normal((L + 1, C, 5 * C)) / np.sqrt(C), device=dev).to(dtype)
    g = torch.tensor(rng.standard_normal((N, M, C)), device=dev).to(dtype)
    cfg = AttentionConfig(heads=H, L=L, r_cut=6.0, box=box)

    def step():
        idx = es.build_neighbors(pos, K, 6.0, seg, box=box, with_distances=False)
        idx.transpose()
        q, k, v = es.project_qk(h, W, L)
        out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
        dq, dk, dv = es.stream_aggregate_backward(g, SavedAttention(q, k, v, pos, idx, out, lse, cfg))
        es.project_qk_backward(h, W, L, dq, dk, dv)
        return idx

    idx = step()
    torch.cuda.synchronize()
    E = int(idx.count.sum().item())
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    F = flops(N, E, L, C, H)
    rec = {"N": N, "pairs": E, "L": L, "C": C, "H": H, "dtype": str(dtype).split(".")[-1], "ms_per_step": round(ms, 4),
           "tflops": round(F / ms / 1e9, 3), "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 3)}
    if cpu:
        from oracle import pyoracle as po
        hh = h.double().cpu().numpy()
        WW = W.double().cpu().numpy()
        gg = g.double().cpu().numpy()
        t0 = time.perf_counter()
        nbr, _, _ = po.build_neighbors(system.pos, K, 6.0, seg_ptr=system.seg_ptr, box=system.box)
        q, k, v = po.project(hh, WW, L)
        P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_EAAS, box=system.box)
        out, lse = po.attn_fwd(P, q, k, v, system.pos, nbr)
        dq, dk, dv = po.attn_bwd(P, q, k, v, system.pos, nbr, out, lse, gg)
        po.project_bwd(hh, WW, L, dq, dk, dv)
        dt = time.perf_counter() - t0
        rec["cpu_oracle_s"] = round(dt, 3)
        rec["cpu_threads"] = po.max_threads()
        rec["gpu_vs_cpu"] = round(dt * 1e3 / ms, 1)
    return rec


def main():
    from paper_2601_16622_b200 import systems as S
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    args = ap.parse_args()
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    for cfg in (int(c) for c in args.configs.split(",")):
        if cfg == 1:
            cases = [(S.config_system(1), 2, 64, 8, True)]
        elif cfg == 3:
            cases = [(S.config_system(3, n_atoms=n), 2, 128, 8, n <= 1000) for n in (1000, 2048, 5000, 10000, 20000)]
        elif cfg == 4:
            cases = [(S.config_system(4), 4, 128, 8, False)]
        elif cfg == 5:
            cases = [(S.config_system(5), 2, 128, 8, False)]
        else:
            continue
        for system, L, C, H, cpu in cases:
            rec = run(system, L, C, H, 64, dt, args.steps, args.warmup, cpu=cpu)
            rec["config"] = cfg
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
