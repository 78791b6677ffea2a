"""CPU-side checks of the C ABI library: it loads, exports every symbol the
header declares, its host-side so3 tables agree with the oracle, and compute
entry points fail loudly without a GPU (no CPU fallback)."""
import ctypes as ct
import math
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "equistream_b200.h")


@pytest.fixture(scope="module")
def eslib():
    from paper_2601_16622_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2601_16622_b200 import build
        build.build()
    return _lib.lib()


def test_exports_match_header(eslib):
    decl = set(re.findall(r"\b(es_[a-z0-9_]+)\s*\(", open(HEADER).read()))
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(eslib, name), f"{name} declared in include/equistream_b200.h but not exported"
    from paper_2601_16622_b200 import _lib
    assert set(_lib.EXPORTS) <= decl


def test_manifest_covers_reference_keys(eslib, oracle):
    text = eslib.es_conventions_manifest().decode()
    keys = {ln.split("=")[0] for ln in text.splitlines() if "=" in ln and not ln.startswith("#")}
    for k in ("m_ordering", "harmonic_normalization", "y00", "complex_basis", "real_basis_change", "l1_value_map",
              "transformation_side", "cg_source", "cg_frobenius_norm_sq_per_path", "cg_odd_path_phase",
              "eaas_reindex_coefficients", "max_degree_tables", "irreps_default_max_degree"):
        assert k in keys  # conventions.hpp:16-36


def test_host_cg_tables_match_oracle(eslib, oracle):
    for l1 in range(5):
        for l2 in range(5):
            for lo in range(abs(l1 - l2), min(l1 + l2, 4) + 1):
                tab = po.cg_real(l1, l2, lo)
                for mo in range(-lo, lo + 1):
                    for m1 in range(-l1, l1 + 1):
                        for m2 in range(-l2, l2 + 1):
                            assert eslib.es_cg_real(l1, m1, l2, m2, lo, mo) == pytest.approx(
                                tab[mo + lo, m1 + l1, m2 + l2], abs=1e-13)


def test_host_reindex_polynomials_match_oracle_rules(eslib, oracle):
    a = (ct.c_double * 5)()
    b = (ct.c_double * 5)()
    for L in range(5):
        for lo in range(L + 1):
            for li in range(L + 1):
                for m in range(-min(lo, li), min(lo, li) + 1):
                    assert eslib.es_reindex_table(L, lo, li, m, a, b) == 0
                    ea = np.zeros(5)
                    eb = np.zeros(5)
                    for lf in range(L + 1):
                        rule = po.reindex_rule(li, lf, lo)
                        if rule is None or m not in rule:
                            continue
                        mi, c = rule[m]
                        c *= math.sqrt((2 * lf + 1) / (4 * math.pi))
                        if (li + lf + lo) % 2 == 0:
                            assert mi == m
                            ea[lf] += c
                        else:
                            assert mi == -m
                            eb[lf] += c
                    np.testing.assert_allclose(np.array(a[:]), ea, atol=1e-13)
                    np.testing.assert_allclose(np.array(b[:]), eb, atol=1e-13)


def test_host_wigner_fit_matches_oracle(eslib, oracle):
    rng = np.random.default_rng(0)
    for _ in range(20):
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        w, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                      [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                      [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
        for l in range(5):
            D = np.zeros((2 * l + 1) ** 2)
            Rc = np.ascontiguousarray(R)
            assert eslib.es_wigner_d_host(l, Rc.ctypes.data_as(ct.POINTER(ct.c_double)),
                                          D.ctypes.data_as(ct.POINTER(ct.c_double))) == 0
            np.testing.assert_allclose(D.reshape(2 * l + 1, -1), po.wigner_d(l, R), atol=1e-12)


def test_invalid_arguments_and_no_cpu_fallback(eslib):
    from paper_2601_16622_b200 import _lib
    d = _lib.AttnDesc()
    d.N, d.K, d.H, d.L, d.C, d.r_cut = 4, 4, 3, 2, 64, 6.0  # C % H != 0
    assert eslib.es_attn_fwd(ct.byref(d), *([None] * 10), 0, None) == _lib.ES_INVALID_ARGUMENT
    assert b"multiple of H" in eslib.es_last_error()
    d.H, d.L = 8, 7
    assert eslib.es_attn_fwd(ct.byref(d), *([None] * 10), 0, None) == _lib.ES_UNSUPPORTED
    d.L, d.bias_mode = 2, 7  # unknown radial-bias form
    assert eslib.es_attn_fwd(ct.byref(d), *([None] * 10), 0, None) == _lib.ES_INVALID_ARGUMENT
    d.bias_mode = 0
    if not eslib.es_device_ok():
        import torch
        import paper_2601_16622_b200 as es
        with pytest.raises(ValueError):
            es.build_neighbors(torch.zeros(4, 3, dtype=torch.float64), 4, 6.0)  # CPU tensor: no fallback


def test_stats_accounting(eslib):
    """OpCounters / stats structure (counters.hpp:11-32):
    algorithmic multiply-adds, forward floating-point scratch independent of K
    (and zero: (mu, z, A) live on chip), backward scratch O(N K H) -- never
    O(N K C) -- and every memory term exactly linear in N."""
    from paper_2601_16622_b200 import api
    cfg = api.AttentionConfig(heads=8, L=2)
    st = api.attn_stats(cfg, 1000, 64, 128, 13600)
    dk, ch, M = 2 * 9 * 128 // 8, 16, 9
    assert st["madds_fwd"] == 13600 * 8 * (dk + ch * M * M)
    assert st["madds_bwd"] == 13600 * 8 * (3 * dk + 2 * ch * M * M)
    assert st["madds_proj_fwd"] == 1000 * 9 * 128 * 5 * 128
    for K in (16, 32, 64):
        assert api.attn_stats(cfg, 1000, K, 128, 13600)["aux_float_bytes_fwd"] == 0
    # backward scratch: no C dependence (C = 64 vs 128), linear in K * H
    b64 = api.attn_stats(cfg, 1000, 64, 64, 0)["aux_float_bytes_bwd"]
    b128 = api.attn_stats(cfg, 1000, 64, 128, 0)["aux_float_bytes_bwd"]
    assert b64 == b128 == 4 * 1000 * 8 + 4 * 1000 * 64 * 8
    # linear in N with R^2 > 0.999 for every byte count
    Ns = np.array([1000, 5000, 20000, 50000, 100000], dtype=np.float64)
    for key in ("aux_float_bytes_bwd", "workspace_bwd_bytes", "workspace_fwd_bytes", "aux_index_bytes"):
        ys = np.array([api.attn_stats(cfg, int(n), 64, 128, 0)[key] for n in Ns], dtype=np.float64)
        if ys.max() == ys.min():  # constant (e.g. no tensor-core tiles without a device): trivially K-free
            continue
        A = np.vstack([Ns, np.ones_like(Ns)]).T
        coef, res, *_ = np.linalg.lstsq(A, ys, rcond=None)
        r2 = 1 - float(((A @ coef - ys) ** 2).sum()) / float(((ys - ys.mean()) ** 2).sum())
        assert r2 > 0.999, (key, r2)
