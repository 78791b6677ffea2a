#!/usr/bin/env python
"""Dense-CG vs EAAS tensor-product microbenchmark on the GPU (
run_tp_bench SPEC.md:449-457, Figure 2: "forward pass time
comparison ... EAAS SO(2)-based tensor product and ... SO(3) tensor product,
l_max=2 and 128 channels").  P independent (feature, direction) pairs; the
value of the attention's path set by the dense Clebsch-Gordan product and by
EAAS (the fused kernels' per-pair device code).  Correctness gate first:
dense == EAAS == the oracle's per-pair operator.  One JSON line per (L, P).

    python bench_tp.py [--L 2,4] [--P 1024,16384,131072] [--C 128]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", default="2,4")
    ap.add_argument("--P", default="1024,16384,131072")
    ap.add_argument("--C", type=int, default=128)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    from paper_2601_16622_b200 import api
    dev = torch.device("cuda")
    for L in (int(x) for x in args.L.split(",")):
        M = (L + 1) ** 2
        dense_m, eaas_m = api.tp_madds(L)
        # correctness gate on 64 pairs against the oracle (checker only, outside any timing)
        from oracle import pyoracle as po
        rng = np.random.default_rng(L)
        v = rng.standard_normal((64, M, args.C)).astype(np.float32)
        r = (rng.standard_normal((64, 3)) * 2.0).astype(np.float32)
        xd = api.tensor_product_pairs(torch.tensor(v, device=dev), torch.tensor(r, device=dev), L, "dense").cpu()
        xe = api.tensor_product_pairs(torch.tensor(v, device=dev), torch.tensor(r, device=dev), L, "eaas").cpu()
        ref = np.stack([po.pair_operator(L, r[p].astype(np.float64), 1, 1e30, 1) @ v[p].astype(np.float64)
                        for p in range(64)])
        sc = np.abs(ref).max()
        gate = {"dense_vs_oracle": float(np.abs(xd.numpy() - ref).max() / sc),
                "eaas_vs_oracle": float(np.abs(xe.numpy() - ref).max() / sc)}
        assert all(e < 1e-4 for e in gate.values()), gate
        for P in (int(x) for x in args.P.split(",")):
            vt = torch.randn((P, M, args.C), device=dev)
            rt = torch.randn((P, 3), device=dev) * 2.0
            t = {}
            for method in ("dense", "eaas"):
                api.tensor_product_pairs(vt, rt, L, method)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(args.iters):
                    api.tensor_product_pairs(vt, rt, L, method)
                b.record()
                torch.cuda.synchronize()
                t[method] = a.elapsed_time(b) / args.iters
            print(json.dumps({"bench": "run_tp_bench", "L_max": L, "C": args.C, "pairs": P,
                              "dense_ms": round(t["dense"], 4), "eaas_ms": round(t["eaas"], 4),
                              "speedup": round(t["dense"] / t["eaas"], 2),
                              "madds_per_pair_channel": {"dense": dense_m, "eaas": eaas_m,
                                                         "ratio": round(dense_m / eaas_m, 2)},
                              "gate_rel_err": gate, "dtype": "fp32"}), flush=True)


if __name__ == "__main__":
    main()
