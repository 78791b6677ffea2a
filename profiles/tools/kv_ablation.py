"""Tensor-core key pass ablation on configs[1] (4096 molecules): the
attn_kv_tc_kernel time with parts of the per-chunk work switched off
(ES_KV_DBG bits: 1 pair math, 2 dOg coupling, 4 D MMA, 8 dV MMA, 16 S MMA,
32 per-head K reload).  Outputs are wrong under the switches -- this only
locates the critical path.

    python profiles/tools/kv_ablation.py [bits ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2601_16622_b200 as es  # noqa: E402
from paper_2601_16622_b200 import systems as S  # noqa: E402
from paper_2601_16622_b200.api import AttentionConfig, SavedAttention  # noqa: E402


def main():
    b = S.molecule_batch(4096, 40, 60, 0)
    L, C, H = 2, 128, 8
    dev = torch.device("cuda")
    pos = torch.tensor(b.pos, device=dev)
    seg = torch.tensor(b.seg_ptr, device=dev)
    h = torch.randn((b.n_atoms, 9, C), device=dev).bfloat16()
    W = (torch.randn((L + 1, C, 5 * C), device=dev) / C ** 0.5).bfloat16()
    idx = es.build_neighbors(pos, 64, 6.0, seg)
    idx.transpose()
    q, k, v = es.project_qk(h, W, L)
    cfg = AttentionConfig(heads=H, L=L)
    out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
    saved = SavedAttention(q, k, v, pos, idx, out, lse, cfg)
    from torch.profiler import ProfilerActivity, profile

    def kv_us():
        es.stream_aggregate_backward(out, saved)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                es.stream_aggregate_backward(out, saved)
            torch.cuda.synchronize()
        tot = {}
        for e in prof.events():
            if e.device_type.name == "CUDA":
                tot[e.name] = tot.get(e.name, 0.0) + e.device_time / 3
        return tot

    var = os.environ.get("ABL_VAR", "ES_KV_DBG")  # ES_DQ_DBG: the dq / dk kernels' switches
    for d in [int(x) for x in (sys.argv[1:] or ["0", "1", "2", "4", "8", "16", "32", "63"])]:
        os.environ[var] = str(d)
        tot = kv_us()
        kv = sum(v for k_, v in tot.items() if "attn_kv_tc" in k_)
        dq = sum(v for k_, v in tot.items() if "attn_dqk_tc_kernel<false>" in k_)
        dk = sum(v for k_, v in tot.items() if "attn_dqk_tc_kernel<true>" in k_)
        print(f"dbg {d:2d}: kv {kv:8.1f} us  dq {dq:7.1f} us  dk {dk:7.1f} us", flush=True)
    os.environ[var] = "0"


if __name__ == "__main__":
    main()
