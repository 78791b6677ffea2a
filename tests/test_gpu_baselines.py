"""The comparison baselines (paper_2601_16622_b200.baselines)
compute the same attention as the fused kernels: edge-materialising (dense
CG per edge) == stream_aggregate (EAAS value), masked dense SDPA ==
stream_aggregate (plain value, phi = 1)."""
import numpy as np
import pytest
import torch

from paper_2601_16622_b200 import systems as S

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).abs().max() / b.abs().max())


@pytest.mark.parametrize("box", [False, True])
def test_edge_materialising_matches_fused(box):
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import baselines
    from paper_2601_16622_b200.api import AttentionConfig
    L, C, H = 2, 64, 8
    if box:
        b = S.periodic_box(220, 4, 3.8, 31)
        pos, bx = torch.tensor(b.pos, device="cuda"), tuple(b.box)
    else:
        pos, bx = torch.tensor(S.gen_fcc_system(300, 3.8, 32), device="cuda"), None
    N = pos.shape[0]
    idx = es.build_neighbors(pos, 64, 6.0, box=bx)
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(N, 9, 2 * C, device="cuda", generator=g)
    k = torch.randn(N, 9, 2 * C, device="cuda", generator=g)
    v = torch.randn(N, 9, C, device="cuda", generator=g)
    out, _ = es.stream_aggregate(q, k, v, pos, idx, AttentionConfig(heads=H, L=L, box=bx))
    ref, peak = baselines.edge_materialising_attention(q, k, v, pos, idx.table, H, L, box=bx, chunk=128)
    assert rel(out, ref) < 1e-4
    assert peak > 0


def test_masked_dense_matches_fused_plain():
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import baselines
    from paper_2601_16622_b200.api import AttentionConfig
    C, H = 64, 8
    pos = torch.tensor(S.gen_fcc_system(400, 3.8, 33), device="cuda")
    idx = es.build_neighbors(pos, 64, 6.0)
    g = torch.Generator(device="cuda").manual_seed(4)
    q = torch.randn(400, 9, 2 * C, device="cuda", generator=g)
    k = torch.randn(400, 9, 2 * C, device="cuda", generator=g)
    v = torch.randn(400, 9, C, device="cuda", generator=g)
    out, _ = es.stream_aggregate(q, k, v, pos, idx, AttentionConfig(heads=H, L=2, value_mode="plain", phi="one"))
    ref = baselines.masked_dense_attention(q, k, v, idx.table, H)
    assert rel(out, ref) < 1e-4


def test_baseline_backwards_match_fused():
    """The backward baselines (autograd through the edge-materialising graph
    and through masked SDPA) equal stream_aggregate_backward (fp32, 1e-4)."""
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import baselines
    from paper_2601_16622_b200.api import AttentionConfig, SavedAttention
    C, H, L = 64, 8, 2
    pos = torch.tensor(S.gen_fcc_system(250, 3.8, 34), device="cuda")
    idx = es.build_neighbors(pos, 64, 6.0)
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(250, 9, 2 * C, device="cuda", generator=g)
    k = torch.randn(250, 9, 2 * C, device="cuda", generator=g)
    v = torch.randn(250, 9, C, device="cuda", generator=g)
    go = torch.randn(250, 9, C, device="cuda", generator=g)
    for vm, phi in (("eaas", "cosine"), ("plain", "one")):
        cfg = AttentionConfig(heads=H, L=L, value_mode=vm, phi=phi)
        out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
        ref = es.stream_aggregate_backward(go, SavedAttention(q, k, v, pos, idx, out, lse, cfg))
        if vm == "eaas":
            fn = lambda a, b_, c: baselines.edge_materialising_attention(a, b_, c, pos, idx.table, H, L, chunk=64)[0]  # noqa: E731
        else:
            fn = lambda a, b_, c: baselines.masked_dense_attention(a, b_, c, idx.table, H)  # noqa: E731
        got = baselines.baseline_backward(fn, q, k, v, go)
        for a_, b_ in zip(got, ref):
            assert rel(a_, b_) < 1e-4, vm
