"""Probe for output rows the backward leaves unwritten: the caching allocator is
filled with NaN first, so any row a kernel skips shows up as non-finite."""
import torch, sys
sys.path.insert(0, ".")
import paper_2601_16622_b200 as es
from paper_2601_16622_b200 import systems as S
from paper_2601_16622_b200.api import AttentionConfig, SavedAttention
import os
dev = torch.device("cuda")
junk = [torch.full((1 << 28,), float("nan"), device=dev) for _ in range(8)]  # 8 GB of NaN, then freed
del junk
b = S.molecule_batch(2048, 40, 60, 11)
pos = torch.tensor(b.pos, device=dev); seg = torch.tensor(b.seg_ptr, device=dev)
g = torch.Generator(device=dev).manual_seed(3)
h = torch.randn((b.n_atoms, 9, 128), device=dev, generator=g).bfloat16()
W = (torch.randn((3, 128, 640), device=dev, generator=g) / 128 ** 0.5).bfloat16()
idx = es.build_neighbors(pos, 64, 6.0, seg); idx.transpose()
q, k, v = es.project_qk(h, W, 2)
cfg = AttentionConfig(heads=8, L=2)
out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
print("out finite", bool(torch.isfinite(out).all()), "lse nan", int(torch.isnan(lse).sum()))
dout = torch.randn(out.shape, device=dev, generator=g).bfloat16()
saved = SavedAttention(q, k, v, pos, idx, out, lse, cfg)
for mode in ("1", "0"):
    os.environ["ES_KV_TC"] = mode
    r = es.stream_aggregate_backward(dout, saved)
    torch.cuda.synchronize()
    for n, a in zip(("dq", "dk", "dv"), r):
        bad = ~torch.isfinite(a.float()).reshape(a.shape[0], -1).all(1)
        print("mode", mode, n, "nonfinite rows", int(bad.sum()), bad.nonzero()[:5].flatten().tolist())
