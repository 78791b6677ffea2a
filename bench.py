#!/usr/bin/env python
"""Benchmark: fused equivariant-attention fwd+bwd TFLOPS & latency on B200.

One "step" = one pass of the hot path over one batch (default: BASELINE.json
configs[1], the SPICE-like batch: 4096 synthetic molecules of U{40..60}
atoms, L_max=2, C=128, H=8, 6 A cutoff):
    neighbour/tile build (+ transposed relation) -> Q/K/V projections ->
    fused EAAS attention forward -> recompute backward -> projection backward
    (dh and dW).
Every launch is a kernel of libequistream_b200.so (plus cub sort/scan and
memsets for the neighbour transpose).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|3|4|5]
    python bench.py --impl reference ...      (the CPU reference arm)

Before any timing, a correctness gate checks the
benched batch itself: neighbour lists of 32 molecules (first and last 16)
bit-exact, out / dq / dk / dv / dh of those molecules against the CPU oracle
(the checker, never the thing timed) at the bf16 tolerance 2e-2, and
equivariance of the whole batch under a random rotation.  A failed gate
aborts the run.

Multi-GPU (one process per GPU; `--gpus N` without torchrun relaunches itself
under torch.distributed.run): configs 2 / 4 shard molecule batches (every rank
its own batch, weak scaling, no data-path collective); configs 3 / 5 shard
the query rows of ONE system (strong scaling: K/V all-gathered once per
layer by NCCL, dk/dv reduce-scattered to their owners).  Timing is CUDA
events, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused equivariant-attention fwd+bwd TFLOPS & latency vs N atoms at 1/2/4/8 B200"
K_, RCUT = 64, 6.0
GATE_TOL = 2e-2  # north_star: bf16-input paths <= 2e-2 with fp32 accumulation
# the forward keeps its scores for the backward only with the tensor-core dk pass (ES_DK_TC=1)
KEEP_SCORES = os.environ.get("ES_DK_TC", "0") == "1"


def flops_per_step(n_atoms: int, n_pairs: int, L: int, C: int, H: int) -> dict:
    """Algorithmic FLOPs (SURVEY.md §8 d)."""
    M = (L + 1) ** 2
    dk = 2 * M * C // H
    ch = C // H
    proj_f = 2 * n_atoms * M * C * (4 * C + C)
    attn_f = n_pairs * H * (2 * dk + 2 * ch * M * M)
    attn_b = n_pairs * H * (6 * dk + 4 * ch * M * M)
    return {"proj_fwd": proj_f, "attn_fwd": attn_f, "attn_bwd": attn_b, "proj_bwd": 2 * proj_f,
            "total": proj_f + attn_f + attn_b + 2 * proj_f}


def call_bytes(n_q: int, n_k: int, n_pairs: int, K: int, s: int, L: int, C: int, H: int) -> dict:
    """Compulsory HBM bytes of each library call (every input read once, every
    output written once).  n_q query rows, n_k key atoms.
    attn_bwd: q, k, v, out (== dout in the bench step: loss = 1/2 ||out||^2,
    read once), lse, pos, nbr + transposed relation in; dq, dk, dv out."""
    M = (L + 1) ** 2
    qk = M * 2 * C * s
    v = M * C * s
    idx = n_q * K * 4
    fwd = n_q * qk + n_k * (qk + v) + n_q * (v + 4 * H) + n_k * 24 + idx
    bwd = n_q * (2 * qk + v + 4 * H) + n_k * (2 * qk + 2 * v + 24) + idx + (n_k + 1) * 4 + n_pairs * 4
    proj_fwd = n_q * (v + 2 * qk + v) + (L + 1) * C * 5 * C * s
    proj_bwd = n_q * (v + 2 * qk + v + v) + (L + 1) * C * 5 * C * (s + 4)
    return {"attn_fwd": fwd, "attn_bwd": bwd, "proj_fwd": proj_fwd, "proj_bwd": proj_bwd}


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "_source": "fallback (B200_PROFILING.md)"}


def fp32_peak() -> dict | None:
    """FP32 CUDA-core peak measured on this GPU now (profiles/tools/fp32_peak.cu)."""
    import ctypes as ct
    so = os.path.join(ROOT, "profiles", "tools", "libfp32peak.so")
    if not os.path.exists(so):
        return None
    lib = ct.CDLL(so)
    lib.es_fp32_peak_tflops.restype = ct.c_double
    lib.es_fp32_peak_tflops.argtypes = [ct.c_int, ct.c_int]
    return {"ffma_tflops": round(lib.es_fp32_peak_tflops(0, 5), 2),
            "ffma2_tflops": round(lib.es_fp32_peak_tflops(1, 5), 2)}


def kernel_times(fn) -> dict:
    """Device time per kernel name (summed) of one call of `fn`, from a
    torch.profiler CUDA trace outside the timed region.  Returns
    {name: (us, launches)} for every CUDA kernel."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    out: dict = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        n = e.name
        us = getattr(e, "device_time", None)
        if us is None:
            us = e.cuda_time
        t, c = out.get(n, (0.0, 0))
        out[n] = (t + float(us), c + 1)
    return out


def short_name(n: str) -> str:
    if "attn_dqk_tc_kernel" in n:
        return "attn_dk_tc" if "<true>" in n else "attn_dq_tc"
    for key in ("attn_fwd_tc", "attn_kv_tc", "attn_pair_geom", "attn_dk_tc", "attn_bwd_q_tc", "attn_bwd_k_tc", "attn_bwd_kv", "attn_dq_tc", "attn_delta",
                "attn_fwd_kernel", "attn_bwd_q_kernel", "proj_fwd_tc", "proj_dh_tc", "proj_dw_tc", "proj_fwd_kernel",
                "proj_bwd", "nbr_segment", "nbr_grid", "tr_sort", "tr_fill", "tr_count", "tc_rowlist", "tc_tiles",
                "tc_mask", "tc_count", "tc_fill", "tc_rowtile", "grid_", "DeviceScan", "DeviceRadix", "nccl"):
        if key in n:
            return key.rstrip("_")
    return n[:60]


def load_traffic():
    """DRAM bytes / tensor-pipe % per launch of the attention kernels from the
    committed ncu --set full capture (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    return json.load(open(p)) if os.path.exists(p) else None


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def wait_live(self, timeout: float = 3.0):
        """Block until nvidia-smi has written its first sample (its start-up takes longer than a short
        timed region), so the samples cover the timed steps."""
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < timeout:
            try:
                if os.path.getsize(self.path) > 0:
                    return
            except OSError:
                pass
            time.sleep(0.02)

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


# ------------------------------------------------------------------ workloads
class Workload:
    """One benchmark configuration on one rank: device inputs, the step (the
    public API calls a user makes), host inputs for the e2e leg."""

    def __init__(self, args, rank: int, world: int, dev):
        import torch

        from paper_2601_16622_b200 import systems
        from paper_2601_16622_b200.api import AttentionConfig
        self.args, self.rank, self.world, self.dev = args, rank, world, dev
        self.dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
        self.L, self.C, self.H = systems.CONFIG_SHAPES[args.config]
        cfgno = args.config
        seed = systems.default_seed(0)
        self.row_sharded = cfgno in (3, 5) and world > 1
        if cfgno in (2, 4):
            seed = seed + 1000003 * rank  # every rank: its own molecule batch
            n_mol = args.molecules if cfgno == 2 else args.molecules_l4
            self.sys = systems.config_system(cfgno, seed, n_mol=n_mol)
        else:
            self.sys = systems.config_system(cfgno, seed, n_atoms=args.atoms)
        self.box = None if self.sys.box is None else tuple(float(b) for b in self.sys.box)
        # scores are recomputed in the backward at every L (keeping them was measured slower at L = 4:
        # key pass 17.1 -> 19.6 ms, profiles/r02e_l4_variants.jsonl)
        self.cfg = AttentionConfig(heads=self.H, L=self.L, r_cut=RCUT, value_mode="eaas", box=self.box)
        N = self.sys.n_atoms
        self.N = N
        M = (self.L + 1) ** 2
        if self.row_sharded:
            from paper_2601_16622_b200.distributed import RowPlan
            self.plan = RowPlan(N, world)
            self.a0, self.a1 = self.plan.rows(rank)
        else:
            self.a0, self.a1 = 0, N
        rng = np.random.default_rng(seed + 17)
        self.h_host = rng.standard_normal((self.a1 - self.a0, M, self.C)).astype(np.float32)
        rng_w = np.random.default_rng(systems.default_seed(0) + 23)  # weights identical on every rank
        self.W_host = (rng_w.standard_normal((self.L + 1, self.C, 5 * self.C)) / np.sqrt(self.C)).astype(np.float32)
        self.pos_host = np.ascontiguousarray(self.sys.pos)
        self.seg_host = None if self.sys.seg_ptr is None else np.ascontiguousarray(self.sys.seg_ptr, dtype=np.int32)
        t = lambda a: torch.tensor(a, device=dev)  # noqa: E731
        self.inputs = [t(self.pos_host), None if self.seg_host is None else t(self.seg_host),
                       t(self.h_host).to(self.dtype), t(self.W_host).to(self.dtype)]
        if self.row_sharded:
            from paper_2601_16622_b200.distributed import CudaBackend, RowShardedAttention
            self.layer = RowShardedAttention(N, CudaBackend(self.cfg), rank, world)

    def describe(self) -> str:
        c = self.args.config
        if c == 2:
            return (f"configs[1] SPICE-like batch: {self.args.molecules} molecules x U{{40..60}} atoms per GPU, "
                    "L_max=2, C=128, H=8, r_cut=6 A, fwd+bwd (neighbours + projections + fused EAAS attention + "
                    "backward; loss = 1/2 ||out||^2 on the device, dout = out)")
        if c == 4:
            return (f"configs[3] OMol25-like batch: {self.args.molecules_l4} molecules x 350 atoms per GPU, L_max=4, "
                    "C=128, H=8, fwd+bwd")
        if c == 3:
            return f"configs[2] single FCC system N={self.N}, L_max=2, C=128, H=8, fwd+bwd, rows sharded over GPUs"
        return (f"configs[4] periodic FCC box N={self.N} (PBC), L_max=2, C=128, H=8, fwd+bwd, query rows sharded "
                "over GPUs with an NCCL all-gather of K/V and reduce-scatter of dk/dv")

    def step(self, pos, seg, h, W):
        """One fwd+bwd pass through the public API; returns (idx, dh, dW)."""
        import paper_2601_16622_b200 as es
        from paper_2601_16622_b200.api import SavedAttention
        if self.row_sharded:
            idx = es.build_neighbors(pos, K_, RCUT, None, box=self.box, with_distances=False,
                                     rows=(self.a0, self.a1))
            out = self.layer.forward(h, W, pos, idx.table)
            dh, dW = self.layer.backward(out)
            return idx, dh, dW
        idx = es.build_neighbors(pos, K_, RCUT, seg, box=self.box, with_distances=False)
        idx.transpose()
        q, k, v = es.project_qk(h, W, self.L)
        out, lse, sc = es.stream_aggregate(q, k, v, pos, idx, self.cfg, return_scores=True) if KEEP_SCORES else \
            (*es.stream_aggregate(q, k, v, pos, idx, self.cfg), None)
        dq, dk, dv = es.stream_aggregate_backward(out, SavedAttention(q, k, v, pos, idx, out, lse, self.cfg,
                                                                      scores=sc))
        dh, dW = es.project_qk_backward(h, W, self.L, dq, dk, dv)
        return idx, dh, dW


# ------------------------------------------------------------------ correctness gate
def rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def random_rotation(seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    qq = rng.standard_normal(4)
    w, x, y, z = qq / np.linalg.norm(qq)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def correctness_gate(wl: Workload) -> dict:
    """the benched batch itself is checked before timing.
    Molecules are independent, so the first and last 16 molecules of the
    4096-molecule batch are compared with the CPU oracle (the checker) run on
    exactly those molecules; equivariance covers the whole batch."""
    import torch

    import paper_2601_16622_b200 as es
    from oracle import pyoracle as po
    from paper_2601_16622_b200.api import SavedAttention, rotate_features
    po.build()
    pos, seg, h, W = wl.inputs
    L, H = wl.L, wl.H
    idx = es.build_neighbors(pos, K_, RCUT, seg, box=wl.box, with_distances=False)
    q, k, v = es.project_qk(h, W, L)
    out, lse = es.stream_aggregate(q, k, v, pos, idx, wl.cfg)
    dq, dk, dv = es.stream_aggregate_backward(out, SavedAttention(q, k, v, pos, idx, out, lse, wl.cfg))
    dh, _ = es.project_qk_backward(h, W, L, dq, dk, dv)
    torch.cuda.synchronize()
    res = {"tol": GATE_TOL}
    seg_h = wl.seg_host
    n_mol = len(seg_h) - 1
    pick = [(0, min(16, n_mol)), (max(0, n_mol - 16), n_mol)]
    hb = h.float().double().cpu().numpy()
    Wb = W.float().double().cpu().numpy()
    errs = {"out": 0.0, "dq": 0.0, "dk": 0.0, "dv": 0.0, "dh": 0.0}
    nbr_ok = True
    mols = 0
    P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_DENSE)
    for m0, m1 in pick:
        a0, a1 = int(seg_h[m0]), int(seg_h[m1])
        lseg = (seg_h[m0:m1 + 1] - a0).astype(np.int32)
        p_ = wl.pos_host[a0:a1]
        nbr_o, _, _ = po.build_neighbors(p_, K_, RCUT, seg_ptr=lseg)
        g_nbr = idx.table[a0:a1].cpu().numpy()
        g_nbr = np.where(g_nbr >= 0, g_nbr - a0, -1)
        nbr_ok &= bool(np.array_equal(g_nbr, nbr_o))
        # the oracle consumes the GPU's own bf16 operands (storage rounding is the input, not the error)
        qo, ko, vo = (x[a0:a1].float().double().cpu().numpy() for x in (q, k, v))
        go = out[a0:a1].float().double().cpu().numpy()
        ro, rl = po.attn_fwd(P, qo, ko, vo, p_, nbr_o)
        rdq, rdk, rdv = po.attn_bwd(P, qo, ko, vo, p_, nbr_o, ro, rl, go)
        rdh, _ = po.project_bwd(hb[a0:a1], Wb, L, rdq, rdk, rdv)
        for name, g, r in (("out", out, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv), ("dh", dh, rdh)):
            errs[name] = max(errs[name], rel(g[a0:a1].float().cpu().numpy(), r))
        mols += m1 - m0
    res["molecules_checked"] = mols
    res["neighbors_bit_exact"] = nbr_ok
    res["rel_err"] = {k_: float(f"{v_:.3g}") for k_, v_ in errs.items()}
    # equivariance of the whole batch: f(R pos, D h) == D f(pos, h), out and dh (bf16 tcgen05 path)
    R = random_rotation(20260117)
    pos_r = pos @ torch.tensor(R.T, device=pos.device)
    h_r = rotate_features(h, L, R)
    idx_r = es.build_neighbors(pos_r.contiguous(), K_, RCUT, seg, box=wl.box, with_distances=False)
    q2, k2, v2 = es.project_qk(h_r, W, L)
    out2, lse2 = es.stream_aggregate(q2, k2, v2, pos_r.contiguous(), idx_r, wl.cfg)
    dq2, dk2, dv2 = es.stream_aggregate_backward(out2, SavedAttention(q2, k2, v2, pos_r.contiguous(), idx_r, out2,
                                                                      lse2, wl.cfg))
    dh2, _ = es.project_qk_backward(h_r, W, L, dq2, dk2, dv2)
    e_out = rel(out2.float().cpu().numpy(), rotate_features(out, L, R).float().cpu().numpy())
    e_dh = rel(dh2.float().cpu().numpy(), rotate_features(dh, L, R).float().cpu().numpy())
    res["equivariance_rel_err"] = {"out": float(f"{e_out:.3g}"), "dh": float(f"{e_dh:.3g}")}
    ok = nbr_ok and all(v_ < GATE_TOL for v_ in errs.values()) and e_out < GATE_TOL and e_dh < GATE_TOL
    res["passed"] = bool(ok)
    return res


# ------------------------------------------------------------------ GPU arm
def time_steps(wl: Workload, steps: int, warmup: int, world: int, sample_clocks: int | None = None):
    import torch
    import torch.distributed as dist
    clk = ClockSampler(sample_clocks) if sample_clocks is not None else None
    if clk:  # live before the warm-up, so it samples through the timed steps
        clk.__enter__()
        clk.wait_live()
    for _ in range(warmup):
        wl.step(*wl.inputs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        wl.step(*wl.inputs)
    e1.record(st)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if world > 1:
        dist.barrier()
    return e0.elapsed_time(e1) / steps, (clk.summary() if clk else None)


def time_call(fn, reps: int = 5) -> float:
    import torch
    st = torch.cuda.current_stream()
    fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def sweep_vs_n(args, dev) -> dict:
    """configs[2]: latency and TFLOP/s vs N (single FCC systems, fwd+bwd, 1 GPU)."""
    import torch
    out = {"N": [], "pairs": [], "ms": [], "tflops": []}
    for n in args.sweep:
        a2 = argparse.Namespace(**vars(args))
        a2.config, a2.atoms = 3, n
        wl = Workload(a2, 0, 1, dev)
        idx, _, _ = wl.step(*wl.inputs)
        torch.cuda.synchronize()
        E = int(idx.count.sum().item())
        ms, _ = time_steps(wl, 10, 3, 1)
        fl = flops_per_step(wl.N, E, wl.L, wl.C, wl.H)["total"]
        out["N"].append(n)
        out["pairs"].append(E)
        out["ms"].append(round(ms, 4))
        out["tflops"].append(round(fl / (ms * 1e-3) / 1e12, 3))
        del wl
        torch.cuda.empty_cache()
    return out


def gpu_arm(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200.api import SavedAttention

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wl = Workload(args, rank, world, dev)
    L, C, H = wl.L, wl.C, wl.H

    gate = None
    if args.config == 2 and not args.no_gate:
        gate = correctness_gate(wl)
        ok = torch.tensor([1 if gate["passed"] else 0], device=dev)
        if world > 1:  # every rank checks its own batch; all abort together (no rank left in a collective)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            if rank == 0:
                print(json.dumps({"metric": METRIC, "error": "correctness gate failed; timing aborted",
                                  "gate": gate}), flush=True)
            if world > 1:
                dist.destroy_process_group()
            sys.exit(3)

    idx, _, _ = wl.step(*wl.inputs)
    torch.cuda.synchronize()
    E = int(idx.count.sum().item())
    n_loc = wl.a1 - wl.a0
    fl = flops_per_step(n_loc, E, L, C, H)
    s_bytes = 2 if wl.dtype == torch.bfloat16 else 4

    ms, clocks = time_steps(wl, args.steps, args.warmup, world, sample_clocks=local_rank)

    # ---- end to end through the public API with HOST buffers (pinned, the
    # user's storage dtype): H2D of every step's inputs (positions, segment
    # table, node features h, weights W) and D2H of its result (dW) inside the
    # timed region; copies on a side stream, double buffered so step s+1's
    # upload overlaps step s's kernels.
    st = torch.cuda.current_stream()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    host = [pin(wl.pos_host), None if wl.seg_host is None else pin(wl.seg_host),
            pin(wl.h_host).to(wl.dtype).pin_memory(), pin(wl.W_host).to(wl.dtype).pin_memory()]
    dW_host = torch.empty((L + 1, C, 5 * C), dtype=torch.float32).pin_memory()
    h2d = sum(x.numel() * x.element_size() for x in host if x is not None)
    d2h = dW_host.numel() * 4
    cs = torch.cuda.Stream(device=dev)
    bufs = [[None if x is None else torch.empty_like(x, device=dev) for x in host] for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]

    def upload(slot):
        with torch.cuda.stream(cs):
            cs.wait_event(freed[slot])
            for d_, h_ in zip(bufs[slot], host):
                if d_ is not None:
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
            _, _, dW = wl.step(*bufs[slot])
            dW_host.copy_(dW, non_blocking=True)
            freed[slot].record(st)

    e2e_run(max(3, args.warmup))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    e2e_run(args.steps)
    b.record(st)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / args.steps

    vals = torch.tensor([ms, e2e_ms, float(fl["total"]), float(n_loc), float(E)], device=dev, dtype=torch.float64)
    if world > 1:
        mx = vals[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = vals[2:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, e2e_ms = float(mx[0]), float(mx[1])
        total_flops, total_atoms, total_pairs = float(tot[0]), int(tot[1]), int(tot[2])
    else:
        total_flops, total_atoms, total_pairs = float(fl["total"]), n_loc, E

    # ---- per-call and per-kernel times (outside the timed region, same stream)
    kt = kernel_times(lambda: wl.step(*wl.inputs))
    launches_per_step = sum(c for n, (_, c) in kt.items() if "es::" in n or "cub::" in n)
    if rank != 0:
        return None
    roof = None
    if not wl.row_sharded:
        pos, seg, h, W = wl.inputs
        q, k, v = es.project_qk(h, W, L)
        idx = es.build_neighbors(pos, K_, RCUT, seg, box=wl.box, with_distances=False)
        idx.transpose()
        fwd = lambda: es.stream_aggregate(q, k, v, pos, idx, wl.cfg, return_scores=KEEP_SCORES)  # noqa: E731
        res = fwd()
        out, lse, sc = res if KEEP_SCORES else (*res, None)
        saved = SavedAttention(q, k, v, pos, idx, out, lse, wl.cfg, scores=sc)
        dq, dk, dv = es.stream_aggregate_backward(out, saved)
        t = {"attn_fwd": time_call(fwd),
             "attn_bwd": time_call(lambda: es.stream_aggregate_backward(out, saved)),
             "proj_fwd": time_call(lambda: es.project_qk(h, W, L)),
             "proj_bwd": time_call(lambda: es.project_qk_backward(h, W, L, dq, dk, dv))}
        kt_bwd = kernel_times(lambda: es.stream_aggregate_backward(out, saved))
        kt_fwd = kernel_times(fwd)
        roof = roofline(wl, t, kt_fwd, kt_bwd, kt, n_loc, E, s_bytes, fl, ms)
    line = {
        "metric": METRIC,
        "value": round(total_flops / (ms * 1e-3) / 1e12, 4),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong" if wl.row_sharded else "weak",
        "vs_baseline": None,
        "dtype": "bf16" if wl.dtype == torch.bfloat16 else "fp32",
        "data": "synthetic (FCC molecules / systems, random features and weights; seeded)",
        "config": {
            "workload": wl.describe(),
            "atoms_per_gpu": n_loc, "pairs_per_gpu": E, "atoms_total": total_atoms, "pairs_total": total_pairs,
            "K": K_, "L_max": L, "channels": C, "heads": H,
            "precision": f"{args.dtype} storage, fp32 accumulation",
            "l2": "inputs exceed L2 (h, q, k, v, dout >= 0.47 GB each at bf16, config 2)",
            "parallelism": (f"rows{world} (query-row slabs, NCCL all-gather K/V + reduce-scatter dk/dv)"
                            if wl.row_sharded else
                            f"dp{world} (molecule batches, no collective)" if args.config in (2, 4) else
                            "one system on one GPU"),
            "latency_ms": round(ms, 4), "flops_per_step_per_gpu": fl,
        },
        "clocks": clocks,
        "e2e": {"value": round(total_flops / (e2e_ms * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
        "kernels_per_step": {short_name(n): {"us": round(t_, 1), "launches": c}
                             for n, (t_, c) in sorted(kt.items(), key=lambda x: -x[1][0])[:14]},
    }
    if gate is not None:
        line["gate"] = gate
    if roof is not None:
        line["roofline"] = roof
    if world == 1 and args.sweep and args.config == 2:
        line["vs_n"] = sweep_vs_n(args, dev)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_molecules, args.cpu_molecules_1t)
    return line


def roofline(wl, t, kt_fwd, kt_bwd, kt_step, n_loc, E, s_bytes, fl, step_ms) -> dict:
    """Roofline of the dominant call, computed on ONE consistent kernel set:
    achieved = algorithmic bytes of the call / CUDA-event time of the same
    call; traffic = ncu DRAM bytes summed over the same call's kernels."""
    peaks = load_peaks()
    by = call_bytes(n_loc, n_loc, E, K_, s_bytes, wl.L, wl.C, wl.H)
    dom = max(t, key=lambda n: t[n])
    kset = kt_bwd if dom == "attn_bwd" else kt_fwd if dom == "attn_fwd" else {}
    achieved = by[dom] / (t[dom] * 1e-3) / 1e9
    tr = load_traffic()
    traffic = None
    tensor_pct = {}
    if tr and kset:
        recs = {short_name(k_): r_ for k_, r_ in tr.get("bytes_per_launch", {}).items()}
        tot, ok = 0.0, True
        for n in kset:
            sn = short_name(n)
            rec = recs.get(sn)
            if rec is None:
                ok = False
                continue
            tot += rec["total"] * kset[n][1]
            if "tensor_pipe_pct" in rec:
                tensor_pct[sn] = rec["tensor_pipe_pct"]
        traffic = tot if ok else None
    flop_key = {"attn_fwd": "attn_fwd", "attn_bwd": "attn_bwd", "proj_fwd": "proj_fwd", "proj_bwd": "proj_bwd"}[dom]
    fp = fp32_peak()
    per_kernel = {}
    step_us = sum(v_[0] for v_ in kt_step.values())
    for n, (us, c) in sorted(kset.items(), key=lambda x: -x[1][0]):
        per_kernel[short_name(n)] = {"us": round(us, 1), "share_of_call": round(us / max(1e-9, sum(
            v_[0] for v_ in kset.values())), 3), "share_of_step": round(us / max(1e-9, step_us), 3)}
    return {
        "kernel": {"attn_bwd": "es_attn_bwd (all its kernels)", "attn_fwd": "es_attn_fwd (all its kernels)",
                   "proj_fwd": "es_project_fwd", "proj_bwd": "es_project_bwd"}[dom],
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
        "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
        "traffic_source": (tr or {}).get("source") if traffic is not None else None,
        "peak_source": peaks["_source"] + " (burst copy bandwidth)",
        "algorithmic_bytes_per_launch": by[dom],
        "call_ms": round(t[dom], 4),
        "achieved_tflops": round(fl[flop_key] / (t[dom] * 1e-3) / 1e12, 3),
        "compute_frac_bf16_dense": round(fl[flop_key] / (t[dom] * 1e-3) / 1e12 / peaks["bf16_tflops"], 4),
        "calls_ms": {k_: round(v_, 4) for k_, v_ in t.items()},
        "calls_frac_hbm": {k_: round(by[k_] / (t[k_] * 1e-3) / 1e9 / peaks["hbm_gbs"], 4) for k_ in t},
        "calls_bytes": by,
        "kernels": per_kernel,
        "tensor_pipe_pct_ncu": tensor_pct or None,
        "fp32_peak_measured": fp,
        # a SIMT key pass (forces / ES_KV_TC=0) computes in fp32 on the CUDA cores: its compute roofline is
        # the FFMA2 peak; the tensor-core key pass is reported against the bf16 peak above
        "compute_frac_fp32_simt": (round(fl[flop_key] / (t[dom] * 1e-3) / 1e12 / fp["ffma2_tflops"], 4)
                                   if fp and fp.get("ffma2_tflops", 0) > 0 and "attn_bwd_kv" in per_kernel
                                   else None),
        "step_frac_hbm": round(sum(by.values()) / (step_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
    }


# ------------------------------------------------------------------ CPU arms
def cpu_sample(n_mol: int, seed: int = 0):
    from oracle import pyoracle as po
    from paper_2601_16622_b200 import systems
    L, C, H = systems.CONFIG_SHAPES[2]
    b = systems.molecule_batch(n_mol, 40, 60, seed)
    N = b.n_atoms
    M = (L + 1) ** 2
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((N, M, C))
    W = rng.standard_normal((L + 1, C, 5 * C)) / np.sqrt(C)
    t0 = time.perf_counter()
    nbr, _, cnt = po.build_neighbors(b.pos, K_, RCUT, seg_ptr=b.seg_ptr)
    q, k, v = po.project(h, W, L)
    P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_EAAS)
    out, lse = po.attn_fwd(P, q, k, v, b.pos, nbr)
    dq, dk, dv = po.attn_bwd(P, q, k, v, b.pos, nbr, out, lse, out)  # loss = 1/2 ||out||^2
    po.project_bwd(h, W, L, dq, dk, dv)
    dt = time.perf_counter() - t0
    E = int(cnt.sum())
    return flops_per_step(N, E, L, C, H)["total"] / dt / 1e12, N, E, dt


def cpu_baseline(n_mol: int, n_mol_1t: int, seed: int = 0) -> dict:
    """The reference CPU algorithm (oracle port: stream_aggregate with per-pair
    EAAS, double accumulators; parallel over atoms, key-centric
    backward) on a bounded sample of the workload -- the first molecules of the
    configs[1] batch, fwd+bwd incl. projections -- at all host threads and at 1."""
    from oracle import pyoracle as po
    po.build()
    cores = po.max_threads()
    v_all, N, E, dt = cpu_sample(n_mol, seed)
    po.set_threads(1)
    v_1, N1, E1, dt1 = cpu_sample(n_mol_1t, seed)
    po.set_threads(cores)
    return {"value": round(v_all, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "value_1thread": round(v_1, 6), "cpu_model": cpu_model(),
            "sample": f"{n_mol} molecules ({N} atoms, {E} pairs) of the configs[1] batch, fwd+bwd, fp64 oracle, "
                      f"{cores} threads: {dt:.2f} s; 1 thread: {n_mol_1t} molecules in {dt1:.2f} s"}


def reference_arm(args, rank: int, world: int):
    if rank != 0:
        return None
    from oracle import pyoracle as po
    po.build()
    cores = po.max_threads()
    vals = []
    warm = args.warmup if args.warmup_ref is None else args.warmup_ref
    for _ in range(min(warm, 1)):
        cpu_sample(args.cpu_molecules)
    info = None
    for _ in range(max(1, min(args.steps, args.ref_steps))):
        v_, N, E, dt = cpu_sample(args.cpu_molecules)
        vals.append(v_)
        info = (N, E, dt)
    val = statistics.mean(vals)
    N, E, dt = info
    return {
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": len(vals), "warmup": min(warm, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp64", "data": "synthetic (FCC molecules, random features/weights; seeded)",
        "config": {"workload": "configs[1] SPICE-like batch (bounded sample, see cpu_baseline.sample)",
                   "L_max": 2, "channels": 128, "heads": 8, "K": K_},
        "cpu_baseline": {"value": round(val, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.cpu_molecules} molecules ({N} atoms, {E} pairs) per step, fwd+bwd, fp64 "
                                   f"oracle port, {cores} threads, {dt:.2f} s per step"},
        "e2e": {"value": round(val, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--molecules", type=int, default=4096)
    ap.add_argument("--molecules-l4", type=int, default=256)
    ap.add_argument("--atoms", type=int, default=None)
    ap.add_argument("--sweep", type=lambda s: [int(x) for x in s.split(",") if x], default=[1000, 2000, 5000,
                                                                                            10000, 20000])
    ap.add_argument("--cpu-molecules", type=int, default=256)
    ap.add_argument("--cpu-molecules-1t", type=int, default=16)
    ap.add_argument("--ref-steps", type=int, default=3)
    ap.add_argument("--warmup-ref", type=int, default=None)  # default: --warmup
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gate", action="store_true")
    args = ap.parse_args()

    in_torchrun = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = reference_arm(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.gpus > 1 and not in_torchrun:
        # one process per GPU: relaunch under torch.distributed.run (127.0.0.1 rendezvous)
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible; "
                             f"run on a node with >= {args.gpus} GPUs\n")
            sys.exit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
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
