"""Run the bf16 parity tests again with the SIMT attention forward kernel forced
(ES_ATTN_TC=0 selects the SIMT kernel; read once per process, hence the subprocess), so a plain
`pytest -m gpu` covers both attention forward kernels (tcgen05 is the default for the
bf16 L=2/C=128/H=8 shape)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_simt_attention_parity():
    env = dict(os.environ, ES_ATTN_TC="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
                        "bf16 or tensor_core or row_sharded"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


@pytest.mark.parametrize("n_mol", [300, 2048])
def test_tensor_core_key_pass_matches_simt_at_size(n_mol, monkeypatch):
    """The tcgen05 key pass (S^T, D = V dOg^T, dV MMAs + tcgen05 dq / dk) against the SIMT key-centric
    pass on the same bf16 molecule batch, at sizes past the oracle tests (15k and 100k atoms, hundreds
    to thousands of key tiles, every tile shape the packer makes): dq, dk, dv agree to the bf16
    tolerance, and every output is finite."""
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import systems as S
    from paper_2601_16622_b200.api import AttentionConfig, SavedAttention
    b = S.molecule_batch(n_mol, 40, 60, 11)
    dev = torch.device("cuda")
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
    dout = torch.randn(out.shape, device=dev, generator=g).bfloat16()
    saved = SavedAttention(q, k, v, pos, idx, out, lse, cfg)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ES_KV_TC", mode)
        res[mode] = [x.float() for x in es.stream_aggregate_backward(dout, saved)]
    torch.cuda.synchronize()
    for name, a, r in zip(("dq", "dk", "dv"), res["1"], res["0"]):
        assert torch.isfinite(a).all(), name
        err = float((a - r).abs().max() / r.abs().max())
        assert err < 2e-2, (name, err)


def test_key_pass_unaligned_lse_takes_simt_pass():
    """The tensor-core key pass bulk-copies lse rows in 16-byte units; an lse buffer that is only
    4-byte aligned (a caller's sliced view) must take the SIMT key pass and give the same gradients."""
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import systems as S
    from paper_2601_16622_b200.api import AttentionConfig, SavedAttention
    b = S.molecule_batch(200, 40, 60, 12)
    dev = torch.device("cuda")
    pos = torch.tensor(b.pos, device=dev)
    g = torch.Generator(device=dev).manual_seed(5)
    h = torch.randn((b.n_atoms, 9, 128), device=dev, generator=g).bfloat16()
    W = (torch.randn((3, 128, 640), device=dev, generator=g) / 128 ** 0.5).bfloat16()
    idx = es.build_neighbors(pos, 64, 6.0, torch.tensor(b.seg_ptr, device=dev))
    q, k, v = es.project_qk(h, W, 2)
    cfg = AttentionConfig(heads=8, L=2)
    out, lse = es.stream_aggregate(q, k, v, pos, idx, cfg)
    dout = torch.randn(out.shape, device=dev, generator=g).bfloat16()
    ref = es.stream_aggregate_backward(dout, SavedAttention(q, k, v, pos, idx, out, lse, cfg))
    buf = torch.empty(lse.numel() + 1, dtype=lse.dtype, device=dev)
    lse_odd = buf[1:].view_as(lse)
    lse_odd.copy_(lse)
    assert lse_odd.data_ptr() % 16 != 0
    got = es.stream_aggregate_backward(dout, SavedAttention(q, k, v, pos, idx, out, lse_odd, cfg))
    torch.cuda.synchronize()
    for name, a_, r_ in zip(("dq", "dk", "dv"), got, ref):
        err = float((a_.float() - r_.float()).abs().max() / r_.float().abs().max())
        assert err < 2e-2, (name, err)
