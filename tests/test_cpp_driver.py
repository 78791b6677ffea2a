"""The C++ header front end (include/equistream/attention/stream_attention.hpp)
compiles with g++ against the C ABI and behaves like the reference (errors as
std::invalid_argument without a device; config-1 parity with a device)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2601_16622_b200 import systems as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    from paper_2601_16622_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2601_16622_b200 import build
        build.build()
    exe = tmp_path / "capi_driver"
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O2", os.path.join(ROOT, "tests", "cpp", "capi_driver.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-L", libdir,
           "-l:libequistream_b200.so", f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)]
    subprocess.check_call(cmd)
    return exe


def _inputs(tmp_path, kind="f32"):
    """config 1 (N=64 FCC, L=2, C=64) in fp32, or a bf16 molecule batch at the
    tensor-core shape (L=2, C=128, H=8)."""
    if kind == "f32":
        L, C, H = 2, 64, 8
        pos, seg = S.gen_fcc_system(64, 3.8, 0), None
    else:
        L, C, H = 2, 128, 8
        b = S.molecule_batch(10, 40, 60, 3)
        pos, seg = b.pos, b.seg_ptr
    N = len(pos)
    h = S.random_features(N, L, C, 0)
    W = S.random_weights(L, C, 0)
    q, k, v = po.project(h, W, L)
    dout = np.random.default_rng(5).standard_normal(v.shape)
    if kind == "bf16":  # the storage rounding the driver applies is the oracle's input
        import torch
        q, k, v, dout = (torch.tensor(x).bfloat16().double().numpy() for x in (q, k, v, dout))
    blob = tmp_path / f"in_{kind}.bin"
    with open(blob, "wb") as f:
        f.write(pos.astype(np.float64).tobytes())
        if seg is not None:
            f.write(np.asarray(seg, np.int32).tobytes())
        for a in (q, k, v, dout):
            f.write(a.astype(np.float32).tobytes())
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    return blob, pos, seg, f32(q), f32(k), f32(v), f32(dout), (N, 0 if seg is None else len(seg) - 1, L, C, H)


def test_cpp_driver_builds_and_reports_errors(tmp_path, oracle):
    exe = _build(tmp_path)
    blob, *_, dims = _inputs(tmp_path)
    out = subprocess.run([str(exe), str(blob), str(tmp_path / "o.bin"), "f32", *map(str, dims)],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "invalid_argument ok" in out.stdout or "OK" in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("kind,tol", [("f32", 1e-5), ("bf16", 2e-2)])
def test_cpp_driver_parity_on_gpu(tmp_path, oracle, kind, tol):
    """The C++ front end end to end (neighbours, transpose, tiles, forward with
    kept scores, backward), elementwise against the oracle: fp32 config 1 and
    the bf16 tensor-core path (tcgen05 forward, dq and dk)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = _build(tmp_path)
    blob, pos, seg, q, k, v, dout, dims = _inputs(tmp_path, kind)
    N, _, L, C, H = dims
    env = dict(os.environ, ES_ATTN_TC="1")
    outp = tmp_path / "o.bin"
    r = subprocess.run([str(exe), str(blob), str(outp), kind, *map(str, dims)], capture_output=True, text=True,
                       env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    M = (L + 1) ** 2
    raw = np.fromfile(outp, dtype=np.float32).astype(np.float64)
    sizes = [N * M * C, N * M * 2 * C, N * M * 2 * C, N * M * C, N * H]
    parts = np.split(raw, np.cumsum(sizes)[:-1])
    out, dq, dk, dv = (p.reshape(N, M, -1) for p in parts[:4])
    lse = parts[4].reshape(N, H)
    nbr, _, _ = po.build_neighbors(pos, 64, 6.0, seg_ptr=seg)
    P = po.AttnProblem(L=L, H=H, value_mode=po.VALUE_DENSE)
    ro, rl = po.attn_fwd(P, q, k, v, pos, nbr)
    rdq, rdk, rdv = po.attn_bwd(P, q, k, v, pos, nbr, ro, rl, dout)

    def rel(a, b):
        return float(np.abs(a - b).max() / np.abs(b).max())

    fin = np.isfinite(rl)
    errs = {"out": rel(out, ro), "lse": rel(lse[fin], rl[fin]), "dq": rel(dq, rdq), "dk": rel(dk, rdk),
            "dv": rel(dv, rdv)}
    assert all(e < tol for e in errs.values()), errs
