"""The sharded layers on the CUDA backend over a real NCCL process group
(world size 1 on the single GPU available here: exercises the NCCL
all_gather_into_tensor / reduce_scatter_tensor / all_to_all_single calls and
the row0 / compact-key plumbing end to end; multi-rank logic is covered by
tests/test_distributed_gloo.py)."""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2601_16622_b200 import systems as S

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("halo", [False, True, "overlap"])
def test_sharded_layer_nccl_world1_matches_layer(nccl_group, halo):
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import distributed as D
    from paper_2601_16622_b200.api import AttentionConfig
    L, C, H = 2, 64, 8
    b = S.periodic_box(200, 4, 3.8, 41)
    pos = torch.tensor(b.pos, device="cuda")
    N = pos.shape[0]
    cfg = AttentionConfig(heads=H, L=L, box=tuple(b.box))
    idx = es.build_neighbors(pos, 64, 6.0, box=b.box)
    h = torch.tensor(S.random_features(N, L, C, 42), device="cuda", dtype=torch.float32)
    W = torch.tensor(S.random_weights(L, C, 42), device="cuda", dtype=torch.float32)
    g = torch.randn(N, 9, C, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
    if halo == "overlap":  # the overlapped path (async NCCL gather / reduce-scatter, local-key interior rows)
        layer = D.RowShardedAttention(N, D.CudaBackend(cfg), 0, 1, overlap="force")
    else:
        layer = (D.HaloShardedAttention if halo else D.RowShardedAttention)(N, D.CudaBackend(cfg), 0, 1)
    out = layer.forward(h, W, pos, idx.table)
    dh, dW = layer.backward(g)
    hr = h.clone().requires_grad_(True)
    Wr = W.clone().requires_grad_(True)
    ref = es.attention_layer(hr, Wr, pos, idx, cfg)
    ref.backward(g)
    rel = lambda a, b_: float((a - b_).abs().max() / b_.abs().max())  # noqa: E731
    assert rel(out, ref.detach()) < 1e-5
    assert rel(dh, hr.grad) < 1e-5
    assert rel(dW, Wr.grad) < 1e-5
