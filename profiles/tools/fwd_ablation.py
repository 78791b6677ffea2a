"""Forward tcgen05 kernel ablation on configs[1] (4096 molecules): time
es_attn_fwd with parts of the per-chunk work switched off (ES_TC_DBG bits:
1 skip Vg math, 2 skip Wt math, 4 skip value MMA, 8 skip S MMA).  Outputs
are wrong under the switches -- this only locates the critical path.

    python profiles/tools/fwd_ablation.py
"""
import os
import sys

import numpy as np
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
    out, lse, sc = es.stream_aggregate(q, k, v, pos, idx, cfg, return_scores=True)
    saved = SavedAttention(q, k, v, pos, idx, out, lse, cfg, scores=sc)
    saved0 = SavedAttention(q, k, v, pos, idx, out, lse, cfg)

    def t(fn, n=5):
        fn()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        return a.elapsed_time(e) / n

    for d in [int(x) for x in (sys.argv[1:] or ["0", "1", "2", "3", "4", "8", "12", "15"])]:
        os.environ["ES_TC_DBG"] = str(d)
        print(f"dbg {d:2d}: fwd {t(lambda: es.stream_aggregate(q, k, v, pos, idx, cfg)):.3f} ms  (keeping scores "
              f"{t(lambda: es.stream_aggregate(q, k, v, pos, idx, cfg, return_scores=True)):.3f} ms)", flush=True)
    os.environ["ES_TC_DBG"] = "0"
    print(f"bwd {t(lambda: es.stream_aggregate_backward(out, saved)):.3f} ms (saved scores), "
          f"{t(lambda: es.stream_aggregate_backward(out, saved0)):.3f} ms (recomputed)")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        es.stream_aggregate(q, k, v, pos, idx, cfg, return_scores=True)
        es.stream_aggregate_backward(out, saved)
        es.stream_aggregate_backward(out, saved0)
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if e.device_type.name == "CUDA" and getattr(e, "device_time_total", 0) > 20:
            print(f"  {getattr(e, 'device_time_total', 0):9.1f} us  {e.key[:90]}")


if __name__ == "__main__":
    main()
