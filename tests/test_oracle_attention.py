"""Oracle attention / neighbour semantics and the
committed reference golden vectors.  CPU only."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2601_16622_b200 import systems as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "so3_ref.npz")


def test_oracle_vs_reference_golden(oracle):
    g = np.load(GOLD)
    for l in range(5):
        Y = np.stack([po.solid_harmonics(l, p) for p in g["points"]])
        np.testing.assert_array_equal(Y, g[f"solid_l{l}"])
    for key in g.files:
        if key.startswith("cg_"):
            l1, l2, lo = (int(c) for c in key[3:])
            np.testing.assert_array_equal(po.cg_real(l1, l2, lo), g[key])
        if key.startswith("tp_") and key.endswith("_out"):
            l1, l2, lo = (int(c) for c in key[3:6])
            out = po.tensor_product_dense(g[key[:6] + "_u"], l1, g[key[:6] + "_v"], l2, lo)
            np.testing.assert_allclose(out, g[key], atol=1e-14)


def _problem(N=64, L=2, C=16, H=4, K=32, seed=0, vm=po.VALUE_DENSE):
    pos = S.gen_fcc_system(N, 3.8, seed)
    nbr, _, _ = po.build_neighbors(pos, K, 6.0)
    h = S.random_features(N, L, C, seed)
    W = S.random_weights(L, C, seed)
    q, k, v = po.project(h, W, L)
    return po.AttnProblem(L=L, H=H, value_mode=vm), pos, nbr, q, k, v


@pytest.mark.parametrize("vm", [po.VALUE_PLAIN, po.VALUE_DENSE, po.VALUE_EAAS])
def test_stream_equals_dense_reference(oracle, vm):
    """Acceptance 5 incl. zero-neighbour and all-padding rows."""
    P, pos, nbr, q, k, v = _problem(vm=vm)
    nbr = nbr.copy()
    nbr[3] = -1            # all-padding row
    nbr[5, 1:] = -1        # single neighbour
    out, lse = po.attn_fwd(P, q, k, v, pos, nbr)
    ref = po.attn_dense_ref(P, q, k, v, pos, nbr)
    np.testing.assert_allclose(out, ref, atol=1e-12 * np.abs(ref).max())
    assert np.all(out[3] == 0) and np.all(np.isneginf(lse[3]))


def test_single_neighbour_and_uniform(oracle):
    P, pos, nbr, q, k, v = _problem(vm=po.VALUE_PLAIN)
    nbr = nbr.copy()
    nbr[7, 1:] = -1
    j = nbr[7, 0]
    out, _ = po.attn_fwd(P, q, k, v, pos, nbr)
    r = np.linalg.norm(pos[j] - pos[7])
    phi = 0.5 * (np.cos(np.pi * r / 6.0) + 1)
    np.testing.assert_allclose(out[7], phi * v[j], rtol=1e-12)


def test_shift_permutation_padding_invariance(oracle):
    P, pos, nbr, q, k, v = _problem()
    out, _ = po.attn_fwd(P, q, k, v, pos, nbr)
    # permuting neighbour order within a row
    rng = np.random.default_rng(0)
    perm = nbr.copy()
    for i in range(len(perm)):
        rng.shuffle(perm[i])
    np.testing.assert_allclose(po.attn_fwd(P, q, k, v, pos, perm)[0], out, atol=1e-12 * np.abs(out).max())
    # extra padding columns
    padded = np.concatenate([nbr, -np.ones((len(nbr), 7), np.int32)], 1)
    np.testing.assert_allclose(po.attn_fwd(P, q, k, v, pos, padded)[0], out, atol=1e-15 * np.abs(out).max())
    # +1e4 score shift: q -> q + c * unit-dk direction on every key? use scale of keys: shift via adding
    # a constant to all keys of a head's first channel with a matching query offset is not a pure shift;
    # instead scale scores through q -> q + t*k-independent term is impossible, so test stability directly:
    big = q * 1e3
    o2, l2 = po.attn_fwd(P, big, k, v, pos, nbr)
    assert np.isfinite(o2).all() and np.isfinite(l2[np.isfinite(l2)]).all()


def test_gradient_finite_differences(oracle):
    """Acceptance 6: N=8, K=4, C=6, step 1e-5, rel < 1e-4."""
    rng = np.random.default_rng(1)
    N, K, L, C, H = 8, 4, 1, 6, 2
    pos = S.gen_fcc_system(N, 3.8, 3)
    nbr, _, _ = po.build_neighbors(pos, K, 6.0)
    M = (L + 1) ** 2
    q = rng.standard_normal((N, M, 2 * C)); k = rng.standard_normal((N, M, 2 * C))
    v = rng.standard_normal((N, M, C)); g = rng.standard_normal((N, M, C))
    for vm in (po.VALUE_PLAIN, po.VALUE_DENSE):
        P = po.AttnProblem(L=L, H=H, value_mode=vm)
        out, lse = po.attn_fwd(P, q, k, v, pos, nbr)
        grads = po.attn_bwd(P, q, k, v, pos, nbr, out, lse, g)

        def f(qq, kk, vv):
            return float((po.attn_dense_ref(P, qq, kk, vv, pos, nbr) * g).sum())

        for which, grad in enumerate(grads):
            arrs = [q, k, v]
            num = np.zeros_like(arrs[which])
            for idx in np.ndindex(num.shape):
                a = [x.copy() for x in arrs]
                a[which][idx] += 1e-5
                fp = f(*a)
                a[which][idx] -= 2e-5
                num[idx] = (fp - f(*a)) / 2e-5
            assert np.abs(num - grad).max() / np.abs(num).max() < 1e-4


def test_backward_trivial_cases(oracle):
    P, pos, nbr, q, k, v = _problem(vm=po.VALUE_PLAIN)
    out, lse = po.attn_fwd(P, q, k, v, pos, nbr)
    z = po.attn_bwd(P, q, k, v, pos, nbr, out, lse, np.zeros_like(out))
    assert all(np.all(x == 0) for x in z)


def test_attention_equivariance(oracle):
    """Acceptance 4 for the full block: rotate inputs == rotate outputs."""
    L, C, H = 2, 8, 2
    pos = S.gen_fcc_system(40, 3.8, 5)
    nbr, _, _ = po.build_neighbors(pos, 64, 6.0)
    h = S.random_features(40, L, C, 5)
    W = S.random_weights(L, C, 5)
    rng = np.random.default_rng(9)
    qq = rng.standard_normal(4); qq /= np.linalg.norm(qq)
    w, x, y, z = qq
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                  [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                  [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
    Dbig = np.zeros(((L + 1) ** 2, (L + 1) ** 2))
    for l in range(L + 1):
        Dbig[l * l:(l + 1) ** 2, l * l:(l + 1) ** 2] = po.wigner_d(l, R)
    rot = lambda f: np.einsum("ab,nbc->nac", Dbig, f)  # noqa: E731
    for vm in (po.VALUE_DENSE, po.VALUE_EAAS):
        P = po.AttnProblem(L=L, H=H, value_mode=vm)
        q, k, v = po.project(h, W, L)
        out, _ = po.attn_fwd(P, q, k, v, pos, nbr)
        q2, k2, v2 = po.project(rot(h), W, L)
        out2, _ = po.attn_fwd(P, q2, k2, v2, pos @ R.T, nbr)
        np.testing.assert_allclose(out2, rot(out), atol=1e-9 * np.abs(out).max())


def _brute_neighbors(pos, K, rc, seg=None, box=None):
    N = len(pos)
    seg = [0, N] if seg is None else seg
    nbr = -np.ones((N, K), np.int32)
    for s in range(len(seg) - 1):
        a0, a1 = seg[s], seg[s + 1]
        P = pos[a0:a1]
        d = P[None, :, :] - P[:, None, :]
        if box is not None:
            d = d - box * np.rint(d / box)
        d2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        for i in range(a1 - a0):
            js = [j for j in range(a1 - a0) if j != i and d2[i, j] < rc * rc]
            js.sort(key=lambda j: (d2[i, j], j))
            js = js[:K]
            nbr[a0 + i, :len(js)] = np.asarray(js, np.int32) + a0
    return nbr


def test_neighbors_match_brute_force(oracle):
    """SPEC.md:431-439 examples + all-pairs oracle, segments and PBC."""
    pos = S.gen_fcc_system(256, 3.8, 0)
    nbr, dist, cnt = po.build_neighbors(pos, 64, 6.0)
    np.testing.assert_array_equal(nbr, _brute_neighbors(pos, 64, 6.0))
    nbr8, _, _ = po.build_neighbors(pos, 8, 6.0)
    np.testing.assert_array_equal(nbr8, _brute_neighbors(pos, 8, 6.0))
    b = S.molecule_batch(6, 20, 40, seed=1)
    nb, _, _ = po.build_neighbors(b.pos, 32, 6.0, seg_ptr=b.seg_ptr)
    np.testing.assert_array_equal(nb, _brute_neighbors(b.pos, 32, 6.0, list(b.seg_ptr)))
    box = S.periodic_box(400, 5, 3.8, 2)
    npb, _, _ = po.build_neighbors(box.pos, 64, 6.0, box=box.box)
    np.testing.assert_array_equal(npb, _brute_neighbors(box.pos, 64, 6.0, box=box.box))
    # two atoms; r_cut below every distance
    two = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    n2, _, c2 = po.build_neighbors(two, 4, 2.0)
    assert n2.tolist() == [[1, -1, -1, -1], [0, -1, -1, -1]]
    n0, _, c0 = po.build_neighbors(pos, 4, 1.0)
    assert (n0 == -1).all()


def test_fcc_geometry(oracle):
    """Acceptance 9 and the SURVEY counts."""
    pos = S.gen_fcc_system(2048, 3.8, 0)
    _, _, cnt = po.build_neighbors(pos, 64, 6.0)
    assert 40 <= cnt.mean() <= 60 and cnt.max() == 54
    _, _, c64 = po.build_neighbors(S.gen_fcc_system(64, 3.8, 0), 64, 6.0)
    assert c64.sum() == 968
    cell = S.gen_fcc_system(4, 3.8, 0, n_cells=1)
    d = np.linalg.norm(cell[:, None] - cell[None], axis=-1)[np.triu_indices(4, 1)]
    np.testing.assert_allclose(d, 3.8 / np.sqrt(2))


def test_tiles_ref_packing_properties():
    """oracle/tiles_ref.py: packed query tiles hold whole segments (a segment
    longer than a tile is split at 128-row boundaries), never exceed 128 rows,
    and cover every row once; uniform tiles are 128-row blocks."""
    from oracle import tiles_ref as TR
    rng = np.random.default_rng(0)
    sizes = rng.integers(20, 300, size=200)
    seg = np.concatenate([[0], np.cumsum(sizes)])
    N = int(seg[-1])
    ts = TR.tile_starts(N, seg)
    assert ts[0] == 0 and ts[-1] == N and all(b > a for a, b in zip(ts, ts[1:]))
    assert all(b - a <= TR.TQ for a, b in zip(ts, ts[1:]))
    cuts = set(ts)
    for a, b in zip(seg[:-1], seg[1:]):
        inner = [c for c in cuts if a < c < b]
        if b - a <= TR.TQ:
            assert not inner or TR.pack_parts(N) > 1  # only a part boundary may cut a short segment
        else:
            assert all((c - a) % TR.TQ == 0 or c - a < TR.TQ for c in inner) or TR.pack_parts(N) > 1
    assert TR.tile_starts(300) == [0, 128, 256, 300]


# ------------------------------------------------------------------ factorized message
def test_translation_coefficients_match_manifest_closed_form(oracle):
    """translation_coefficients: the least-squares weights of
    R^l(a+b) = sum_u w(l,u) (R^u(a) x R^{l-u}(b))^l equal the closed form of the
    reference manifest (conventions.hpp:32-34); l=1 is vector additivity."""
    for l in range(5):
        w = oracle.translation_coefficients(l)
        ref = np.array([oracle.translation_weight(l, u) for u in range(l + 1)])
        np.testing.assert_allclose(w, ref, rtol=1e-10, atol=1e-12)
    rng = np.random.default_rng(0)
    for _ in range(200):  # l = 2 reconstruction on random (a, b)
        a, b = rng.standard_normal(3), rng.standard_normal(3)
        rec = sum(oracle.translation_weight(2, u) * oracle.tensor_product_dense(
            oracle.solid_harmonics(u, a), u, oracle.solid_harmonics(2 - u, b), 2 - u, 2).ravel() for u in range(3))
        assert np.abs(rec - oracle.solid_harmonics(2, a + b)).max() < 1e-10


def _msg_case(n, L, C, H, seed):
    pos = S.gen_fcc_system(n, 3.8, seed)
    nbr, _, _ = po.build_neighbors(pos, 32, 6.0)
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((n, (L + 1) ** 2, C))
    alpha = rng.random((n, 32, H))
    return pos, nbr, h, alpha


@pytest.mark.parametrize("L", [1, 2])
def test_factorized_equals_edge_centric(oracle, L):
    """factorized_message == edge_centric_message < 1e-9, also
    after translating the whole system by |t| = 100 and 1000 (the binomial
    expansion's stress test), with and without recentring."""
    pos, nbr, h, alpha = _msg_case(24, L, 8, 2, L)
    ref = oracle.edge_message(pos, h, nbr, alpha, L)
    scale = np.abs(ref).max()
    got = oracle.factorized_message(pos, h, nbr, alpha, L)
    assert np.abs(got - ref).max() < 1e-9 * scale
    for t in (100.0, 1000.0):
        shift = np.array([0.6, -0.48, 0.64]) * t
        ref_t = oracle.edge_message(pos + shift, h, nbr, alpha, L)
        assert np.abs(ref_t - ref).max() < 1e-9 * scale  # edge-centric is translation invariant
        got_c = oracle.factorized_message(pos + shift, h, nbr, alpha, L)  # recentred at the centroid
        assert np.abs(got_c - ref).max() < 1e-9 * scale
        if t == 100.0:  # absolute coordinates (no recentring): conditioning grows like |t|^(2L)
            got_abs = oracle.factorized_message(pos + shift, h, nbr, alpha, L, origin=np.zeros(3))
            assert np.abs(got_abs - ref).max() < 1e-6 * scale
