"""ctypes front-end to the CPU oracle (oracle/esoracle.c) and to the
reference-built library (oracle/_ref/libesref.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
the cpu_baseline / ``--impl reference`` legs of bench.py -- never by the
product package, which has no CPU fallback.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libesoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libesref.so")

_dp = ct.POINTER(ct.c_double)
_ip = ct.POINTER(ct.c_int)


def build(force: bool = False) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    src = os.path.join(HERE, "esoracle.c")
    if force or not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    if force or not os.path.exists(REF_SO):
        subprocess.check_call([os.path.join(HERE, "build_ref.sh")])


_lib = None
_ref = None


def lib() -> ct.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ct.CDLL(ORACLE_SO)
        L.eso_factorial.restype = ct.c_double
        L.eso_complex_cg.restype = ct.c_double
        L.eso_wigner_6j.restype = ct.c_double
        L.eso_on_axis_solid_harmonic.restype = ct.c_double
        L.eso_on_axis_solid_harmonic.argtypes = [ct.c_int, ct.c_double]
        L.eso_build_neighbors.argtypes = [ct.c_int, _dp, ct.c_int, _ip, _dp, ct.c_int, ct.c_double, _ip, _dp, _ip]
        L.eso_apply_reindex.argtypes = [ct.c_int, ct.c_int, ct.c_int, _dp, ct.c_int, ct.c_double, _dp]
        L.eso_pair_operator.argtypes = [ct.c_int, ct.c_int, ct.c_double, ct.c_int, _dp, _dp]
        i = ct.c_int
        L.eso_solid_harmonics.argtypes = [i, _dp, _dp]
        L.eso_cg_real.argtypes = [i, i, i, _dp]
        L.eso_wigner_d.argtypes = [i, _dp, _dp]
        L.eso_eaas_tp.argtypes = [_dp, i, i, _dp, i, i, _dp, _dp]
        L.eso_tensor_product_dense.argtypes = [_dp, i, i, _dp, i, i, i, _dp]
        L.eso_reindex_rule.argtypes = [i, i, i, _ip, _dp]
        L.eso_complex_cg.argtypes = [i] * 6
        L.eso_wigner_6j.argtypes = [i] * 6
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> ct.CDLL:
    global _ref
    if _ref is None:
        R = ct.CDLL(REF_SO)
        for f in ("esref_on_axis", "esref_complex_cg", "esref_wigner_6j", "esref_factorial"):
            getattr(R, f).restype = ct.c_double
        R.esref_on_axis.argtypes = [ct.c_int, ct.c_double]
        R.esref_tensor_product_dense.restype = ct.c_longlong
        _ref = R
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _ip_(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def _c(a, dtype=np.float64) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- so3
def solid_harmonics(l: int, r) -> np.ndarray:
    out = np.zeros(2 * l + 1)
    lib().eso_solid_harmonics(l, _p(_c(r)), _p(out))
    return out


def on_axis(l: int, rn: float) -> float:
    return lib().eso_on_axis_solid_harmonic(l, rn)


def complex_cg(j1, m1, j2, m2, J, M) -> float:
    return lib().eso_complex_cg(j1, m1, j2, m2, J, M)


def wigner_6j(*j) -> float:
    return lib().eso_wigner_6j(*j)


def cg_real(l1: int, l2: int, lo: int) -> np.ndarray | None:
    """[2lo+1][2l1+1][2l2+1] real CG table (clebsch.hpp:179), None on triangle violation."""
    out = np.zeros((2 * lo + 1) * (2 * l1 + 1) * (2 * l2 + 1))
    rc = lib().eso_cg_real(l1, l2, lo, _p(out))
    if rc == -1:
        return None
    if rc != 0:
        raise RuntimeError("cg_real: imaginary residue")
    return out.reshape(2 * lo + 1, 2 * l1 + 1, 2 * l2 + 1)


def wigner_d(l: int, R) -> np.ndarray:
    out = np.zeros((2 * l + 1) ** 2)
    lib().eso_wigner_d(l, _p(_c(R)), _p(out))
    return out.reshape(2 * l + 1, 2 * l + 1)


def alignment_rotation(r) -> np.ndarray:
    out = np.zeros(9)
    rc = lib().eso_alignment_rotation(_p(_c(r)), _p(out))
    if rc != 0:
        raise ValueError("alignment_rotation: degenerate direction")
    return out.reshape(3, 3)


def tensor_product_dense(u, l1, v, l2, lo) -> np.ndarray | None:
    """u [2l1+1][C1], v [2l2+1][C2] (C1==C2 or broadcast 1)."""
    l1, l2, lo = int(l1), int(l2), int(lo)
    u = _c(u).reshape(2 * l1 + 1, -1)
    v = _c(v).reshape(2 * l2 + 1, -1)
    C = max(u.shape[1], v.shape[1])
    out = np.zeros((2 * lo + 1, C))
    rc = lib().eso_tensor_product_dense(_p(u), l1, u.shape[1], _p(v), l2, v.shape[1], lo, _p(out))
    return None if rc == -1 else out


def reindex_rule(li, lf, lo):
    src = np.zeros(2 * lo + 1, dtype=np.int32)
    coef = np.zeros(2 * lo + 1)
    n = lib().eso_reindex_rule(li, lf, lo, _ip_(src), _p(coef))
    if n < 0:
        return None
    return {mo - lo: (int(src[mo]), float(coef[mo])) for mo in range(2 * lo + 1) if src[mo] != -1000}


def eaas_tp(h, li, r, lf, lo, R=None) -> np.ndarray:
    li, lf, lo = int(li), int(lf), int(lo)
    h = _c(h).reshape(2 * li + 1, -1)
    out = np.zeros((2 * lo + 1, h.shape[1]))
    Rp = _p(_c(R)) if R is not None else None
    rc = lib().eso_eaas_tp(_p(h), li, h.shape[1], _p(_c(r)), lf, lo, Rp, _p(out))
    if rc != 0:
        raise ValueError("eaas_tp: triangle violation")
    return out


def pair_operator(L, r, value_mode=1, r_cut=6.0, phi_mode=0) -> np.ndarray:
    M = (L + 1) ** 2
    T = np.zeros(M * M)
    lib().eso_pair_operator(L, value_mode, r_cut, phi_mode, _p(_c(r)), _p(T))
    return T.reshape(M, M)


# ---------------------------------------------------------------- neighbours
def build_neighbors(pos, K: int, r_cut: float, seg_ptr=None, box=None):
    """(nbr [N][K] int32 sentinel -1, dist [N][K] f64, count [N] int32)."""
    pos = _c(pos).reshape(-1, 3)
    N = pos.shape[0]
    nbr = np.zeros((N, K), dtype=np.int32)
    dist = np.zeros((N, K))
    cnt = np.zeros(N, dtype=np.int32)
    sp = None if seg_ptr is None else _c(seg_ptr, np.int32)
    bx = None if box is None else _c(box)
    rc = lib().eso_build_neighbors(N, _p(pos), 0 if sp is None else len(sp) - 1,
                                   None if sp is None else _ip_(sp), None if bx is None else _p(bx),
                                   K, float(r_cut), _ip_(nbr), _p(dist), _ip_(cnt))
    if rc != 0:
        raise RuntimeError("build_neighbors: candidate overflow")
    return nbr, dist, cnt


# ---------------------------------------------------------------- attention
VALUE_PLAIN, VALUE_DENSE, VALUE_EAAS = 0, 1, 2


class _Desc(ct.Structure):
    _fields_ = [("N", ct.c_int), ("K", ct.c_int), ("H", ct.c_int), ("L", ct.c_int), ("Dq", ct.c_int),
                ("Cv", ct.c_int), ("r_cut", ct.c_double), ("value_mode", ct.c_int), ("phi_mode", ct.c_int),
                ("box", _dp), ("bias_mode", ct.c_int), ("bias", ct.c_double * 3)]


@dataclass
class AttnProblem:
    L: int
    H: int
    r_cut: float = 6.0
    value_mode: int = VALUE_DENSE
    phi_mode: int = 0
    box: np.ndarray | None = None
    bias: tuple | None = None  # b(r) = b0 + b1 r + b2 r^2; None: b == 0

    def desc(self, N, K, Dq, Cv):
        self._box = None if self.box is None else _c(self.box)
        b = (0.0, 0.0, 0.0) if self.bias is None else tuple(float(x) for x in self.bias) + (0.0,) * (3 - len(self.bias))
        return _Desc(N, K, self.H, self.L, Dq, Cv, self.r_cut, self.value_mode, self.phi_mode,
                     None if self._box is None else _p(self._box), 0 if self.bias is None else 1,
                     (ct.c_double * 3)(*b))


def project(h, W, L):
    """h [N][M][C], W [L+1][C][2Dq+Cv] with Dq = 2C, Cv = C -> (q, k, v)."""
    h = _c(h)
    W = _c(W)
    N, M, C = h.shape
    Wc = W.shape[2]
    Cv = C
    Dq = (Wc - Cv) // 2
    q = np.zeros((N, M, Dq)); k = np.zeros((N, M, Dq)); v = np.zeros((N, M, Cv))
    lib().eso_project(N, L, C, Dq, Cv, _p(h), _p(W), _p(q), _p(k), _p(v))
    return q, k, v


def project_bwd(h, W, L, dq, dk, dv, want_dW=True):
    h = _c(h); W = _c(W)
    N, M, C = h.shape
    Dq = dq.shape[2]; Cv = dv.shape[2]
    dh = np.zeros_like(h)
    dW = np.zeros_like(W) if want_dW else None
    lib().eso_project_bwd(N, L, C, Dq, Cv, _p(h), _p(W), _p(_c(dq)), _p(_c(dk)), _p(_c(dv)), _p(dh),
                          _p(dW) if want_dW else None)
    return dh, dW


def attn_fwd(prob: AttnProblem, q, k, v, pos, nbr):
    q, k, v, pos = _c(q), _c(k), _c(v), _c(pos)
    nbr = _c(nbr, np.int32)
    N, M, Dq = q.shape
    Cv = v.shape[2]
    d = prob.desc(N, nbr.shape[1], Dq, Cv)
    out = np.zeros((N, M, Cv)); lse = np.zeros((N, prob.H))
    lib().eso_attn_fwd(ct.byref(d), _p(q), _p(k), _p(v), _p(pos), _ip_(nbr), _p(out), _p(lse))
    return out, lse


def attn_dense_ref(prob: AttnProblem, q, k, v, pos, nbr):
    q, k, v, pos = _c(q), _c(k), _c(v), _c(pos)
    nbr = _c(nbr, np.int32)
    N, M, Dq = q.shape
    Cv = v.shape[2]
    d = prob.desc(N, nbr.shape[1], Dq, Cv)
    out = np.zeros((N, M, Cv))
    lib().eso_attn_dense_ref(ct.byref(d), _p(q), _p(k), _p(v), _p(pos), _ip_(nbr), _p(out))
    return out


def attn_bwd(prob: AttnProblem, q, k, v, pos, nbr, out, lse, dout):
    q, k, v, pos, out, lse, dout = (_c(a) for a in (q, k, v, pos, out, lse, dout))
    nbr = _c(nbr, np.int32)
    N, M, Dq = q.shape
    Cv = v.shape[2]
    d = prob.desc(N, nbr.shape[1], Dq, Cv)
    dq = np.zeros_like(q); dk = np.zeros_like(k); dv = np.zeros_like(v)
    lib().eso_attn_bwd(ct.byref(d), _p(q), _p(k), _p(v), _p(pos), _ip_(nbr), _p(out), _p(lse), _p(dout),
                       _p(dq), _p(dk), _p(dv))
    return dq, dk, dv


def max_threads() -> int:
    return lib().eso_max_threads()


def set_threads(n: int) -> None:
    lib().eso_set_threads(n)


# ---------------------------------------------------------------- fixtures
def default_seed(fallback: int = 0) -> int:
    """EQUISTREAM_SEED env fallback (rng.hpp:14-22)."""
    try:
        return int(os.environ.get("EQUISTREAM_SEED", fallback))
    except ValueError:
        return fallback


# ------------------------------------------------------------------ factorized message
def translation_weight(l: int, u: int) -> float:
    """Closed form printed by the reference manifest (conventions.hpp:32-34)."""
    f = lib().eso_translation_weight
    f.restype = ct.c_double
    f.argtypes = [ct.c_int, ct.c_int]
    return float(f(l, u))


def translation_coefficients(l: int) -> np.ndarray:
    """Least-squares weights w[u] of R^l(a+b) = sum_u w[u] (R^u(a) x R^{l-u}(b))^l."""
    w = np.zeros(l + 1)
    assert lib().eso_translation_coefficients(int(l), _p(w)) == 0
    return w


def recouple(li, u, lb, lf, lo) -> np.ndarray:
    c = np.zeros(9)
    lib().eso_recouple(int(li), int(u), int(lb), int(lf), int(lo), _p(c))
    return c


def edge_message(pos, h, nbr, alpha, L):
    """edge_centric_message: m_i = sum_j alpha_ij sum_paths (h_j (x) R^lf(r_j - r_i))^lo."""
    pos, h, alpha = _c(pos), _c(h), _c(alpha)
    nbr = _c(nbr, np.int32)
    N, K = nbr.shape
    H = alpha.shape[2]
    C = h.shape[2]
    out = np.zeros_like(h)
    lib().eso_edge_message(N, K, H, int(L), C, _p(pos), _p(h), nbr.ctypes.data_as(_ip), _p(alpha), _p(out))
    return out


def factorized_message(pos, h, nbr, alpha, L, origin=None):
    """factorized_message (Eq. 5); origin defaults to the centroid."""
    pos, h, alpha = _c(pos), _c(h), _c(alpha)
    nbr = _c(nbr, np.int32)
    N, K = nbr.shape
    H = alpha.shape[2]
    C = h.shape[2]
    o = _c(pos.mean(axis=0) if origin is None else np.asarray(origin, np.float64))
    out = np.zeros_like(h)
    lib().eso_factorized_message(N, K, H, int(L), C, _p(pos), _p(o), _p(h), nbr.ctypes.data_as(_ip), _p(alpha),
                                 _p(out))
    return out
