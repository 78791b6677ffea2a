#!/usr/bin/env python
"""The paper's comparison (Fig. 1-3) on the B200: forward
latency and peak memory of the fused EAAS attention (this library) against
the edge-materialising formulation (dense CG per edge, PyTorch) and masked
dense SDPA (PyTorch), on config 3 systems (N = 1k..20k, L=2, C=128, H=8,
6 A cutoff) and the config 2 molecule batch.  One JSON line per (method, N).

    python bench_baselines.py [--sizes 1000,2000,5000,10000,20000] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, (torch.cuda.max_memory_allocated() - base) / 1e9


def run(name, pos, seg, reps, dense_ok):
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import baselines
    from paper_2601_16622_b200.api import AttentionConfig
    L, C, H = 2, 128, 8
    N = pos.shape[0]
    idx = es.build_neighbors(pos, 64, 6.0, seg)
    E = int(idx.count.sum().item())
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(N, 9, 2 * C, device="cuda", generator=g).bfloat16()
    k = torch.randn(N, 9, 2 * C, device="cuda", generator=g).bfloat16()
    v = torch.randn(N, 9, C, device="cuda", generator=g).bfloat16()
    cfg = AttentionConfig(heads=H, L=L)
    rows = []
    ms, gb = timed(lambda: es.stream_aggregate(q, k, v, pos, idx, cfg), reps)
    rows.append({"method": "fused_eaas (this library, bf16)", "ms": round(ms, 4), "peak_gb": round(gb, 3)})
    ms, gb = timed(lambda: baselines.edge_materialising_attention(q, k, v, pos, idx.table, H, L, chunk=8192), reps)
    rows.append({"method": "edge_materialising_dense_cg (torch, fp32 math)", "ms": round(ms, 4),
                 "peak_gb": round(gb, 3)})
    if dense_ok:
        ms, gb = timed(lambda: baselines.masked_dense_attention(q, k, v, idx.table, H), reps)
        rows.append({"method": "masked_dense_sdpa (torch, bf16, plain values)", "ms": round(ms, 4),
                     "peak_gb": round(gb, 3)})
    for r in rows:
        r.update({"system": name, "N": N, "pairs": E, "L": L, "C": C, "H": H, "pass": "forward"})
        print(json.dumps(r), flush=True)
    # forward + backward (the baselines by autograd through their materialised graphs)
    from paper_2601_16622_b200.api import SavedAttention
    go = torch.randn(N, 9, C, device="cuda", generator=g).bfloat16()

    def fused_fb():
        out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
        es.stream_aggregate_backward(go, SavedAttention(q, k, v, pos, idx, out, lse, cfg))

    bw = [("fused_eaas (this library, bf16)", fused_fb)]
    if N <= 20000:  # the per-edge graph of the whole system is kept for the backward
        bw.append(("edge_materialising_dense_cg (torch autograd)", lambda: baselines.baseline_backward(
            lambda a, b_, c: baselines.edge_materialising_attention(a, b_, c, pos, idx.table, H, L, chunk=8192)[0],
            q, k, v, go)))
    if dense_ok:
        bw.append(("masked_dense_sdpa (torch autograd, plain values)", lambda: baselines.baseline_backward(
            lambda a, b_, c: baselines.masked_dense_attention(a, b_, c, idx.table, H), q, k, v, go)))
    for mname, fn in bw:
        try:
            ms, gb = timed(fn, reps)
            r = {"method": mname, "ms": round(ms, 4), "peak_gb": round(gb, 3)}
        except torch.cuda.OutOfMemoryError:
            torch.cuda.empty_cache()
            r = {"method": mname, "error": "OOM"}
        r.update({"system": name, "N": N, "pairs": E, "L": L, "C": C, "H": H, "pass": "forward+backward"})
        print(json.dumps(r), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1000,2000,5000,10000,20000")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--molecules", type=int, default=4096)
    args = ap.parse_args()
    from paper_2601_16622_b200 import systems as S
    for n in [int(x) for x in args.sizes.split(",") if x]:
        pos = torch.tensor(S.gen_fcc_system(n, 3.8, 0), device="cuda")
        run(f"config3 fcc N={n}", pos, None, args.reps, dense_ok=n <= 20000)
    if args.molecules:
        b = S.molecule_batch(args.molecules, 40, 60, 0)
        run(f"config2 {args.molecules} molecules", torch.tensor(b.pos, device="cuda"),
            torch.tensor(b.seg_ptr, device="cuda"), args.reps, dense_ok=False)


if __name__ == "__main__":
    main()
