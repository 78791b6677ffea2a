"""The tile structures the tensor-core kernels walk (es_attn_tiles_build:
query tiles, tile-skip mask -> chunk lists, per-row (chunk, key mask) lists,
ascending-j slot order and its inverse; key-side lists of the dk pass) are
bit-exact against the NumPy restatement in oracle/tiles_ref.py (north_star:
"bit-exact neighbour/tile index lists"; VERDICT r1 missing #3)."""
import ctypes as ct

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from oracle import tiles_ref as TR
from paper_2601_16622_b200 import systems as S

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]


def _cases():
    return {
        "batch_2parts": lambda: (lambda b: (b.pos, b.seg_ptr, None, 64))(S.molecule_batch(100, 40, 60, 4)),
        "batch_long_segments": lambda: (lambda b: (b.pos, b.seg_ptr, None, 64))(S.molecule_batch(8, 100, 300, 5)),
        "bulk_uniform": lambda: (S.gen_fcc_system(3000, 3.8, 6), None, None, 64),
        "bulk_K16_asymmetric": lambda: (S.gen_fcc_system(2000, 3.8, 7), None, None, 16),
        "pbc": lambda: (lambda b: (b.pos, None, b.box, 64))(S.periodic_box(2500, 9, 3.8, 8)),
    }


@pytest.mark.parametrize("case", list(_cases()))
def test_tile_lists_bit_exact(case, monkeypatch):
    monkeypatch.setenv("ES_DK_TC", "1")  # the buffer also carries the key-side lists
    monkeypatch.setenv("ES_ATTN_TC", "1")
    import paper_2601_16622_b200 as es
    from paper_2601_16622_b200 import _lib
    from paper_2601_16622_b200.api import AttentionConfig
    pos, seg, box, K = _cases()[case]()
    N = len(pos)
    tp = torch.tensor(pos, device="cuda")
    ts = None if seg is None else torch.tensor(seg, device="cuda")
    idx = es.build_neighbors(tp, K, 6.0, ts, box)
    cfg = AttentionConfig(heads=8, L=2, box=None if box is None else tuple(box))
    d = cfg.desc(N, K, 128, torch.bfloat16)
    buf = idx.tiles(d)
    assert buf is not None
    lay = _lib.TilesLayout()
    _lib.check(_lib.lib().es_attn_tiles_layout_query(ct.byref(d), ct.byref(lay)), "layout")
    torch.cuda.synchronize()
    raw = buf.cpu().numpy()
    nbr = idx.table.cpu().numpy()
    ref_nbr, _, _ = po.build_neighbors(pos, K, 6.0, seg_ptr=seg, box=box)
    assert np.array_equal(nbr, ref_nbr)

    def arr(off, n, dt=np.int32):
        return raw[off:off + n * np.dtype(dt).itemsize].view(dt)

    # ---- query side
    q = lay.query
    ref = TR.build(nbr, seg)
    nt = len(ref["tstart"]) - 1
    tstart = arr(q.tstart, q.ntiles + 1)
    np.testing.assert_array_equal(tstart[:nt + 1], ref["tstart"])
    assert np.all(tstart[nt:] == N)
    np.testing.assert_array_equal(arr(q.rtile, N), ref["rtile"])
    cptr = arr(q.cptr, q.ntiles + 1)
    np.testing.assert_array_equal(cptr[:nt + 1], ref["cptr"])
    assert np.all(cptr[nt:] == ref["cptr"][-1])  # surplus tiles: empty lists
    clist = arr(q.clist, int(ref["cptr"][-1]))
    for t in range(nt):
        assert list(clist[cptr[t]:cptr[t + 1]]) == ref["clist"][t]
    rl = arr(q.rowlist, N * K, np.uint32).reshape(N, K)
    slots = arr(q.slots, N * K).reshape(N, K)
    rank = arr(q.rank_of, N * K).reshape(N, K)
    for i in range(N):
        n_ent = int(np.argmax(ref["rowlist"][i] == 0xFFFF0000)) if (ref["rowlist"][i] == 0xFFFF0000).any() else K
        upto = min(K, n_ent + 1)
        np.testing.assert_array_equal(rl[i, :upto], ref["rowlist"][i, :upto])
        nv = int((nbr[i] >= 0).sum())
        np.testing.assert_array_equal(slots[i, :nv], ref["slots"][i, :nv])
        vs = np.nonzero(nbr[i] >= 0)[0]
        np.testing.assert_array_equal(rank[i, vs], ref["rank_of"][i, vs])

    # ---- key side (dk pass)
    k = lay.key
    assert k.ntiles > 0
    rev_ptr, rev_pair = (x.cpu().numpy() for x in idx.transpose())
    kref = TR.build_keys(nbr, rev_ptr, rev_pair, seg)
    nt = len(kref["tstart"]) - 1
    tstart = arr(k.tstart, k.ntiles + 1)
    np.testing.assert_array_equal(tstart[:nt + 1], kref["tstart"])
    cptr = arr(k.cptr, k.ntiles + 1)
    np.testing.assert_array_equal(cptr[:nt + 1], kref["cptr"])
    clist = arr(k.clist, int(kref["cptr"][-1]))
    for t in range(nt):
        assert list(clist[cptr[t]:cptr[t + 1]]) == kref["clist"][t]
    krl = arr(k.rowlist, int(rev_ptr[-1]), np.uint32)
    for j in range(N):
        e0 = int(rev_ptr[j])
        ent = kref["rowlist"][j]
        np.testing.assert_array_equal(krl[e0:e0 + len(ent)], ent)
