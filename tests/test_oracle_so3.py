"""Oracle (CPU, double) vs the reference's own so3 code and the SPEC's
known answers (SURVEY.md §4 known-answer table).
CPU only."""
import math

import numpy as np
import pytest

from oracle import pyoracle as po


def _rot(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


# ------------------------------------------------- pinned against the reference headers
def test_harmonics_match_reference(oracle, ref):
    rng = np.random.default_rng(0)
    for _ in range(100):
        r = rng.standard_normal(3) * rng.uniform(0.1, 5)
        for l in range(9):
            b = np.zeros(2 * l + 1)
            assert ref.esref_solid_harmonics(l, po._p(po._c(r)), po._p(b)) == 0
            np.testing.assert_array_equal(po.solid_harmonics(l, r), b)  # bit-identical recursion


def test_harmonics_match_reference_legendre_oracle(oracle, ref):
    """proj/tests/support/legendre_oracle.hpp: independent theta/phi evaluation."""
    rng = np.random.default_rng(1)
    for _ in range(100):
        u = rng.standard_normal(3)
        u /= np.linalg.norm(u)
        for l in range(9):
            b = np.zeros(2 * l + 1)
            ref.esref_legendre_real_sph(l, po._p(po._c(u)), po._p(b))
            np.testing.assert_allclose(po.solid_harmonics(l, u), b, atol=1e-13)


def test_cg_and_6j_match_reference(oracle, ref):
    for l1 in range(5):
        for l2 in range(5):
            for lo in range(abs(l1 - l2), min(l1 + l2, 4) + 1):
                a = po.cg_real(l1, l2, lo)
                b = np.zeros(a.size)
                assert ref.esref_cg_real(l1, l2, lo, po._p(b)) == 0
                np.testing.assert_array_equal(a.ravel(), b)
    for j in [(1, 1, 1, 1, 1, 1), (2, 1, 1, 1, 2, 2), (2, 2, 2, 2, 2, 2), (0, 2, 2, 1, 2, 2), (3, 2, 1, 2, 3, 2)]:
        assert po.wigner_6j(*j) == pytest.approx(ref.esref_wigner_6j(*j), abs=1e-15)


def test_dense_tensor_product_matches_reference(oracle, ref):
    rng = np.random.default_rng(2)
    for l1 in range(5):
        for l2 in range(5):
            for lo in range(abs(l1 - l2), min(l1 + l2, 4) + 1):
                u = rng.standard_normal((2 * l1 + 1, 3))
                v = rng.standard_normal((2 * l2 + 1, 3))
                a = po.tensor_product_dense(u, l1, v, l2, lo)
                b = np.zeros((2 * lo + 1, 3))
                madds = ref.esref_tensor_product_dense(po._p(po._c(u)), l1, 3, po._p(po._c(v)), l2, 3, lo, po._p(b))
                assert madds == 3 * (2 * l1 + 1) * (2 * l2 + 1) * (2 * lo + 1)  # tensor_product.hpp:44-47
                np.testing.assert_allclose(a, b, atol=1e-14)


def test_reference_wigner_defect_F3(oracle, ref):
    """The shipped wigner_d equals the true D of S R^T S; the oracle
    D satisfies the convention anchor (wigner.hpp:19-20)."""
    rng = np.random.default_rng(3)
    S = np.diag([1.0, -1.0, 1.0])
    for _ in range(10):
        R = _rot(rng)
        for l in range(1, 5):
            b = np.zeros((2 * l + 1) ** 2)
            ref.esref_wigner_d(l, po._p(po._c(R)), po._p(b))
            np.testing.assert_allclose(b.reshape(2 * l + 1, -1), po.wigner_d(l, S @ R.T @ S), atol=1e-12)


def test_manifest_keys(oracle, ref):
    import ctypes
    buf = ctypes.create_string_buffer(4096)
    n = ref.esref_conventions_manifest(buf, 4096)
    assert n > 0
    text = buf.value.decode()
    assert "m_ordering=ascending_-l_to_l" in text and "cg_odd_path_phase=-i" in text


# ------------------------------------------------- SPEC known answers
def test_known_answers(oracle):
    assert po.solid_harmonics(0, [0.3, 0.1, 0.2])[0] == pytest.approx(0.28209479177387814)
    assert po.complex_cg(1, 0, 1, 0, 0, 0) == pytest.approx(-1 / math.sqrt(3), abs=1e-15)
    assert po.complex_cg(1, 1, 1, 0, 1, 0) == 0.0  # M != m1+m2
    assert po.complex_cg(3, 0, 0, 0, 3, 0) == pytest.approx(1.0)
    assert po.wigner_6j(1, 1, 1, 1, 1, 1) == pytest.approx(1 / 6)
    assert po.cg_real(0, 0, 0)[0, 0, 0] == pytest.approx(1.0)
    assert po.cg_real(1, 1, 1)[1, 1, 1] == 0.0
    assert po.cg_real(1, 2, 4) is None
    # l=1 value map sqrt(3/4pi) (y, z, -x)  (conventions.hpp:23)
    r = np.array([0.3, -1.2, 0.7])
    np.testing.assert_allclose(po.solid_harmonics(1, r), math.sqrt(3 / (4 * math.pi)) * np.array([r[1], r[2], -r[0]]),
                               atol=1e-15)
    # Frobenius norm^2 = 2 lo + 1 per path (conventions.hpp:27)
    for (a, b, c) in [(1, 1, 2), (2, 2, 2), (2, 1, 3), (4, 4, 4)]:
        assert (po.cg_real(a, b, c) ** 2).sum() == pytest.approx(2 * c + 1)


def test_harmonic_identities(oracle):
    rng = np.random.default_rng(4)
    for _ in range(100):
        R = _rot(rng)
        r = rng.standard_normal(3)
        for l in range(5):
            D = po.wigner_d(l, R)
            np.testing.assert_allclose(po.solid_harmonics(l, R @ r), D @ po.solid_harmonics(l, r), atol=1e-10)
            np.testing.assert_allclose(D @ D.T, np.eye(2 * l + 1), atol=1e-10)
        s = rng.uniform(0.1, 3)
        for l in range(5):
            np.testing.assert_allclose(po.solid_harmonics(l, s * r), s ** l * po.solid_harmonics(l, r), rtol=1e-12,
                                       atol=1e-14)
    R1, R2 = _rot(rng), _rot(rng)
    for l in range(5):
        np.testing.assert_allclose(po.wigner_d(l, R1 @ R2), po.wigner_d(l, R1) @ po.wigner_d(l, R2), atol=1e-10)
    assert np.abs(po.solid_harmonics(2, np.zeros(3))).max() == 0.0


def test_pole_sparsity(oracle):
    """Acceptance 1: Lemma 1 on 1000 random r, l <= 4."""
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(1000):
        r = rng.standard_normal(3) * 3
        R = po.alignment_rotation(r)
        np.testing.assert_allclose(R @ r, [0, 0, np.linalg.norm(r)], atol=1e-10 * np.linalg.norm(r))
        for l in range(5):
            y = po.solid_harmonics(l, R @ r)
            worst = max(worst, np.abs(np.delete(y, l)).max() if l else 0.0)
    assert worst < 1e-12 * 3 ** 4


def test_reindex_rules_structure(oracle):
    """Acceptance 3 + parity rule."""
    assert po.reindex_rule(1, 1, 0) == {0: (0, pytest.approx(-1 / math.sqrt(3)))}
    r111 = po.reindex_rule(1, 1, 1)
    assert 0 not in r111 and r111[-1][0] == 1 and r111[1][0] == -1
    total = 0
    for li in range(5):
        for lf in range(5):
            for lo in range(abs(li - lf), min(li + lf, 4) + 1):
                rule = po.reindex_rule(li, lf, lo)
                total += len(rule)
                for mo, (mi, c) in rule.items():
                    assert mi == (mo if (li + lf + lo) % 2 == 0 else -mo)
                    # exactly the non-zero m_f = 0 column of the dense table
                    tab = po.cg_real(li, lf, lo)
                    assert c == pytest.approx(tab[mo + lo, mi + li, lf])
    assert total == 272  # 65 paths with all l <= 4 carry 272 non-zeros


def test_eaas_exactness(oracle):
    """Acceptance 2, reduced draw count for CI: EAAS == dense."""
    rng = np.random.default_rng(6)
    worst = 0.0
    for _ in range(2000):
        li, lf, lo = (int(x) for x in rng.integers(0, 5, 3))
        if not (abs(li - lf) <= lo <= li + lf):
            continue
        h = rng.standard_normal((2 * li + 1, 2))
        r = rng.standard_normal(3) * rng.uniform(0.5, 3)
        a = po.eaas_tp(h, li, r, lf, lo)
        b = po.tensor_product_dense(h, li, po.solid_harmonics(lf, r)[:, None], lf, lo)
        worst = max(worst, np.abs(a - b).max() / max(1.0, np.abs(b).max()))
    assert worst < 1e-10


def test_eaas_gauge_independence_and_poles(oracle):
    rng = np.random.default_rng(7)
    for r in ([0, 0, 5.0], [0, 0, -1.0], [1e-9, 0, -2.0], rng.standard_normal(3)):
        r = np.asarray(r, float)
        R0 = po.alignment_rotation(r)
        g = rng.uniform(0, 2 * np.pi)
        Rz = np.array([[np.cos(g), -np.sin(g), 0], [np.sin(g), np.cos(g), 0], [0, 0, 1]])
        for (li, lf, lo) in [(1, 1, 1), (2, 2, 2), (2, 1, 3), (3, 2, 1)]:
            h = rng.standard_normal((2 * li + 1, 3))
            a = po.eaas_tp(h, li, r, lf, lo, R0)
            b = po.eaas_tp(h, li, r, lf, lo, Rz @ R0)
            np.testing.assert_allclose(a, b, atol=1e-10)
    np.testing.assert_allclose(po.alignment_rotation([0, 0, 5.0]), np.eye(3))


def test_madd_ratio(oracle):
    """Acceptance 8 op-count substitute: dense/EAAS >= 3 per l_f >= 1 path at l_max = 2."""
    for li in range(3):
        for lf in range(1, 3):
            for lo in range(abs(li - lf), min(li + lf, 2) + 1):
                dense = (2 * li + 1) * (2 * lf + 1) * (2 * lo + 1)
                sparse = len(po.reindex_rule(li, lf, lo))
                assert dense / max(sparse, 1) >= 3
