"""Isolation probe for the intermittent tensor-core backward mismatch (DESIGN 8.0):
runs the GPU parity suite in-process (the state that triggers it), then the
2048-molecule backward twice per key-pass mode and reports pairwise max
differences -- a mode that disagrees with itself is nondeterministic."""
import os
import sys

import pytest
import torch

sys.path.insert(0, os.getcwd())
pytest.main(["-q", "-m", "gpu", "-x", "tests/test_gpu_parity.py", "-p", "no:cacheprovider"])
import paper_2601_16622_b200 as es
from paper_2601_16622_b200 import systems as S
from paper_2601_16622_b200.api import AttentionConfig, SavedAttention

dev = torch.device("cuda")
b = S.molecule_batch(2048, 40, 60, 11)
pos = torch.tensor(b.pos, device=dev)
seg = torch.tensor(b.seg_ptr, device=dev)
g = torch.Generator(device=dev).manual_seed(3)
h = torch.randn((b.n_atoms, 9, 128), device=dev, generator=g).bfloat16()
W = (torch.randn((3, 128, 640), device=dev, generator=g) / 128 ** 0.5).bfloat16()
idx = es.build_neighbors(pos, 64, 6.0, seg)
idx.transpose()
q, k, v = es.project_qk(h, W, 2)
cfg = AttentionConfig(heads=8, L=2)
out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
out2, _ = es.stream_aggregate(q, k, v, pos, idx, cfg)
print("fwd repeat maxdiff", float((out.float() - out2.float()).abs().max()))
dout = torch.randn(out.shape, device=dev, generator=g).bfloat16()
saved = SavedAttention(q, k, v, pos, idx, out, lse, cfg)
res = {}
for mode in ("1", "0"):
    os.environ["ES_KV_TC"] = mode
    res[mode] = [[x.float() for x in es.stream_aggregate_backward(dout, saved)] for _ in range(2)]
torch.cuda.synchronize()


def d(a, b):
    return [round(float((x - y).abs().max() / y.abs().max()), 5) for x, y in zip(a, b)]


print("tc  vs tc  (dq, dk, dv):", d(res["1"][0], res["1"][1]))
print("simt vs simt (dq, dk, dv):", d(res["0"][0], res["0"][1]))
print("tc  vs simt (dq, dk, dv):", d(res["1"][0], res["0"][0]), d(res["1"][1], res["0"][1]))
