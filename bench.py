#!/usr/bin/env python
"""Benchmark: fused equivariant-attention fwd+bwd TFLOPS & latency on B200.

One "step" = one pass of the hot path over one batch (BASELINE.json
configs[1], the SPICE-like batch: 4096 synthetic molecules of U{40..60}
atoms, L_max=2, C=128, H=8, 6 A cutoff):
    neighbour/tile build (+ transposed relation) -> Q/K/V projections ->
    fused EAAS attention forward -> recompute backward -> projection backward
    (dh and dW).
Every launch is a kernel of libequistream_b200.so (plus cub sort/scan and
memsets for the neighbour transpose).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype bf16|fp32]
    python bench.py --impl reference ...      (the CPU reference arm)

Multi-GPU (torchrun, one process per GPU): the molecule batch is the unit;
every rank processes its own 4096-molecule batch (weak scaling, no data-path
collective -- molecules are independent); timing is CUDA events, max over
ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused equivariant-attention fwd+bwd TFLOPS & latency vs N atoms at 1/2/4/8 B200"
L_, C_, H_, K_, RCUT = 2, 128, 8, 64, 6.0


def flops_per_step(n_atoms: int, n_pairs: int, L=L_, C=C_, H=H_) -> dict:
    """Algorithmic FLOPs (SURVEY.md §8 d)."""
    M = (L + 1) ** 2
    dk = 2 * M * C // H
    ch = C // H
    proj_f = 2 * n_atoms * M * C * (4 * C + C)
    attn_f = n_pairs * H * (2 * dk + 2 * ch * M * M)
    attn_b = n_pairs * H * (6 * dk + 4 * ch * M * M)
    return {"proj_fwd": proj_f, "attn_fwd": attn_f, "attn_bwd": attn_b, "proj_bwd": 2 * proj_f,
            "total": proj_f + attn_f + attn_b + 2 * proj_f}


def attn_bytes(n_atoms: int, n_pairs: int, K: int, s: int, L=L_, C=C_, H=H_) -> dict:
    """Compulsory HBM bytes per launch of the attention kernels (each input
    read once, each output written once)."""
    M = (L + 1) ** 2
    qk = n_atoms * M * 2 * C * s
    v = n_atoms * M * C * s
    fwd = 2 * qk + v + v + n_atoms * (24 + 4 * H) + n_atoms * K * 4
    # kv pass: q, k, v, dout, lse, delta, pos, rev lists in; dk, dv, dscore out
    kv = 2 * qk + v + v + (qk + v) + n_atoms * (24 + 8 * H) + 2 * n_pairs * 4 + n_pairs * H * 4
    return {"attn_fwd": fwd, "attn_bwd_kv": kv}


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "_source": "fallback (B200_PROFILING.md)"}


def count_launches(fn) -> int:
    """Kernels of libequistream_b200.so (incl. the cub scans it launches)
    in one call of `fn`, from a torch.profiler CUDA trace taken outside the
    timed region."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    return sum(1 for n in names if "es::" in n or "cub::" in n)


def load_traffic():
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    the attention kernels from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    return json.load(open(p)) if os.path.exists(p) else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in open(self.path):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ GPU arm
def gpu_arm(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import api, systems
    from paper_2601_16622_b200.api import AttentionConfig, SavedAttention

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    seed = systems.default_seed(0) + 1000003 * rank  # each rank: its own molecule batch
    batch = systems.molecule_batch(args.molecules, 40, 60, seed)
    N = batch.n_atoms
    M = (L_ + 1) ** 2
    rng = np.random.default_rng(seed)
    h_host = rng.standard_normal((N, M, C_)).astype(np.float32)
    W_host = (rng.standard_normal((L_ + 1, C_, 5 * C_)) / np.sqrt(C_)).astype(np.float32)
    cfg = AttentionConfig(heads=H_, L=L_, r_cut=RCUT, value_mode="eaas")

    pos = torch.tensor(batch.pos, device=dev)
    seg = torch.tensor(batch.seg_ptr, device=dev)
    h = torch.tensor(h_host, device=dev).to(dtype)
    W = torch.tensor(W_host, device=dev).to(dtype)

    # One training-like pass: loss = 1/2 ||out||^2 on the device, so the
    # gradient seed is dout = out (no upstream gradient crosses PCIe); the
    # step's result is dW (what an optimizer consumes).
    def step(pos, seg, h, W):
        idx = es.build_neighbors(pos, K_, RCUT, seg, with_distances=False)
        idx.transpose()
        q, k, v = es.project_qk(h, W, L_)
        out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
        dq, dk, dv = es.stream_aggregate_backward(out, SavedAttention(q, k, v, pos, idx, out, lse, cfg))
        dh, dW = es.project_qk_backward(h, W, L_, dq, dk, dv)
        return idx, dh, dW

    idx, _, _ = step(pos, seg, h, W)
    torch.cuda.synchronize()
    E = int(idx.count.sum().item())
    fl = flops_per_step(N, E)
    s_bytes = 2 if dtype == torch.bfloat16 else 4
    by = attn_bytes(N, E, K_, s_bytes)

    for _ in range(args.warmup):
        step(pos, seg, h, W)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(st)
        for _ in range(args.steps):
            step(pos, seg, h, W)
        e1.record(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.summary()

    # per-kernel share: time the attention kernels alone with events (same stream)
    q, k, v = es.project_qk(h, W, L_)
    idx = es.build_neighbors(pos, K_, RCUT, seg, with_distances=False)
    rev = idx.transpose()
    out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
    torch.cuda.synchronize()
    t = {}
    for name, fn in (("attn_fwd", lambda: es.stream_aggregate(q, k, v, pos, idx, cfg)),
                     ("attn_bwd", lambda: es.stream_aggregate_backward(
                         out, SavedAttention(q, k, v, pos, idx, out, lse, cfg))),
                     ("proj_fwd", lambda: es.project_qk(h, W, L_)),
                     ("neighbors", lambda: es.build_neighbors(pos, K_, RCUT, seg, with_distances=False))):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(3):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        t[name] = a.elapsed_time(b) / 3

    # end to end through the public API with HOST buffers (pinned, the
    # user's storage dtype): H2D of every step's inputs (positions, segment
    # table, node features h, weights W) and D2H of its result (dW) inside
    # the timed region; copies run on a side stream, double buffered so step
    # s+1's upload overlaps step s's kernels.
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hp = pin(h_host).to(dtype).pin_memory()
    Wp = pin(W_host).to(dtype).pin_memory()
    posp, segp = pin(batch.pos), pin(batch.seg_ptr)
    dW_host = torch.empty((L_ + 1, C_, 5 * C_), dtype=torch.float32).pin_memory()
    h2d = sum(x.numel() * x.element_size() for x in (hp, Wp, posp, segp))
    d2h = dW_host.numel() * 4
    cs = torch.cuda.Stream(device=dev)
    bufs = [[torch.empty_like(x, device=dev) for x in (posp, segp, hp, Wp)] for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]

    def upload(slot):
        with torch.cuda.stream(cs):
            cs.wait_event(freed[slot])
            for d_, h_ in zip(bufs[slot], (posp, segp, hp, Wp)):
                d_.copy_(h_, non_blocking=True)
            copied[slot].record(cs)

    def e2e_run(n):
        for b_ in range(2):
            freed[b_].record(st)
        upload(0)
        for s_ in range(n):
            slot = s_ % 2
            if s_ + 1 < n:
                upload(1 - slot)
            st.wait_event(copied[slot])
            _, _, dW = step(*bufs[slot])
            dW_host.copy_(dW, non_blocking=True)
            freed[slot].record(st)

    e2e_run(max(2, args.warmup))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    e2e_run(args.steps)
    b.record(st)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / args.steps

    vals = torch.tensor([ms, e2e_ms, float(fl["total"]), float(N), float(E)], device=dev, dtype=torch.float64)
    if world > 1:
        mx = vals[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = vals[2:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, e2e_ms = float(mx[0]), float(mx[1])
        total_flops, total_atoms, total_pairs = float(tot[0]), int(tot[1]), int(tot[2])
    else:
        total_flops, total_atoms, total_pairs = float(fl["total"]), N, E
    if rank != 0:
        return None
    peaks = load_peaks()
    traffic_src = load_traffic()
    dom = max(("attn_fwd", "attn_bwd"), key=lambda n: t[n])
    dom_kernels = ["attn_fwd_tc_kernel"] if dom == "attn_fwd" else ["attn_delta_kernel", "attn_bwd_kv_kernel",
                                                                    "attn_dq_tc_kernel"]
    traffic = None
    if traffic_src and all(k_ in traffic_src["bytes_per_launch"] for k_ in dom_kernels):
        traffic = sum(traffic_src["bytes_per_launch"][k_]["total"] for k_ in dom_kernels)
    dom_bytes = by["attn_fwd"] if dom == "attn_fwd" else by["attn_bwd_kv"]
    achieved = dom_bytes / (t[dom] * 1e-3) / 1e9
    dom_flops = fl["attn_fwd"] if dom == "attn_fwd" else fl["attn_bwd"]
    launches_per_step = count_launches(lambda: step(pos, seg, h, W))
    line = {
        "metric": METRIC,
        "value": round(total_flops / (ms * 1e-3) / 1e12, 4),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16" if dtype == torch.bfloat16 else "fp32",
        "data": "synthetic (FCC molecules, random features/weights; seeded)",
        "config": {
            "workload": "configs[1] SPICE-like batch: 4096 molecules x U{40..60} atoms per GPU, L_max=2, C=128, "
                        "H=8, r_cut=6 A, fwd+bwd (neighbours + projections + fused EAAS attention + backward; "
                        "loss = 1/2 ||out||^2 on the device, dout = out)",
            "molecules_per_gpu": args.molecules, "atoms_per_gpu": N, "pairs_per_gpu": E,
            "atoms_total": total_atoms, "pairs_total": total_pairs, "K": K_, "L_max": L_, "channels": C_,
            "heads": H_, "precision": f"{args.dtype} storage, fp32 accumulation",
            "l2": "inputs exceed L2 (h, q, k, v, dout >= 0.47 GB each at bf16)",
            "parallelism": f"dp{world} (molecule batches, no collective)",
            "latency_ms": round(ms, 4), "flops_per_step_per_gpu": fl,
        },
        "roofline": {
            "kernel": "attn_fwd_tc_kernel (tcgen05)" if dom == "attn_fwd" else
                      "attn_bwd (delta + bwd_kv SIMT + dq tcgen05)",
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
            "traffic_source": traffic_src["source"] if traffic is not None else None,
            "peak_source": peaks["_source"],
            "algorithmic_bytes_per_launch": dom_bytes,
            "achieved_tflops": round(dom_flops / (t[dom] * 1e-3) / 1e12, 3),
            "kernel_ms": {k_: round(v_, 4) for k_, v_ in t.items()},
            "note": "forward: tcgen05 kernel (S = Q K^T and O += Wt Vg on the tensor cores, per-pair geometry "
                    "on CUDA cores); backward: key-centric fp32 SIMT kernel (per-pair EAAS adjoint; dk, dv, "
                    "dscore) + tcgen05 dq = dS K",
        },
        "clocks": clocks,
        "e2e": {"value": round(total_flops / (e2e_ms * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_molecules, threads=None)
    return line


# ------------------------------------------------------------------ CPU arms
def cpu_baseline(n_mol: int, threads: int | None, seed: int = 0) -> dict:
    """The reference CPU algorithm (oracle port: stream_aggregate with per-pair
    EAAS, double accumulators) on a bounded sample of the
    workload: the first n_mol molecules of the batch, fwd+bwd incl. projections."""
    from oracle import pyoracle as po
    from paper_2601_16622_b200 import systems

    po.build()
    if threads:
        po.set_threads(threads)
    cores = po.max_threads()
    b = systems.molecule_batch(n_mol, 40, 60, seed)
    N = b.n_atoms
    M = (L_ + 1) ** 2
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((N, M, C_))
    W = rng.standard_normal((L_ + 1, C_, 5 * C_)) / np.sqrt(C_)
    t0 = time.perf_counter()
    nbr, _, cnt = po.build_neighbors(b.pos, K_, RCUT, seg_ptr=b.seg_ptr)
    q, k, v = po.project(h, W, L_)
    P = po.AttnProblem(L=L_, H=H_, value_mode=po.VALUE_EAAS)
    out, lse = po.attn_fwd(P, q, k, v, b.pos, nbr)
    dq, dk, dv = po.attn_bwd(P, q, k, v, b.pos, nbr, out, lse, out)  # loss = 1/2 ||out||^2
    po.project_bwd(h, W, L_, dq, dk, dv)
    dt = time.perf_counter() - t0
    fl = flops_per_step(N, int(cnt.sum()))
    return {"value": round(fl["total"] / dt / 1e12, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "sample": f"{n_mol} molecules ({N} atoms, {int(cnt.sum())} pairs) of the configs[1] batch, fwd+bwd, "
                      f"fp64 oracle, {dt:.2f} s"}


def reference_arm(args, rank: int, world: int):
    if rank != 0:
        return None
    steps = []
    warm = args.warmup if args.warmup_ref is None else args.warmup_ref
    for _ in range(warm):
        cpu_baseline(args.cpu_molecules, threads=None)
    for _ in range(max(1, min(args.steps, args.ref_steps))):
        steps.append(cpu_baseline(args.cpu_molecules, threads=None))
    val = statistics.mean(s["value"] for s in steps)
    base = steps[0]
    return {
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": len(steps), "warmup": warm, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp64", "data": "synthetic (FCC molecules, random features/weights; seeded)",
        "config": {"workload": "configs[1] SPICE-like batch (bounded sample, see cpu_baseline.sample)",
                   "L_max": L_, "channels": C_, "heads": H_, "K": K_},
        "cpu_baseline": {**base, "value": round(val, 6)},
        "e2e": {"value": round(val, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--molecules", type=int, default=4096)
    ap.add_argument("--cpu-molecules", type=int, default=32)
    ap.add_argument("--ref-steps", type=int, default=3)
    ap.add_argument("--warmup-ref", type=int, default=None)  # default: --warmup
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = reference_arm(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = gpu_arm(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
