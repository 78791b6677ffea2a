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


def _inputs(tmp_path):
    L, C, N = 2, 64, 64
    pos = S.gen_fcc_system(N, 3.8, 0)
    h = S.random_features(N, L, C, 0)
    W = S.random_weights(L, C, 0)
    q, k, v = po.project(h, W, L)
    blob = tmp_path / "in.bin"
    with open(blob, "wb") as f:
        f.write(pos.astype(np.float64).tobytes())
        for a in (q, k, v):
            f.write(a.astype(np.float32).tobytes())
    return blob, pos, q.astype(np.float32).astype(np.float64), k.astype(np.float32).astype(np.float64), \
        v.astype(np.float32).astype(np.float64)


def test_cpp_driver_builds_and_reports_errors(tmp_path, oracle):
    exe = _build(tmp_path)
    blob, *_ = _inputs(tmp_path)
    out = subprocess.run([str(exe), str(blob)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "invalid_argument ok" in out.stdout or "CHECKSUM" in out.stdout


@pytest.mark.gpu
def test_cpp_driver_parity_on_gpu(tmp_path, oracle):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = _build(tmp_path)
    blob, pos, q, k, v = _inputs(tmp_path)
    out = subprocess.run([str(exe), str(blob)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    s, s2 = (float(x) for x in out.stdout.split("CHECKSUM")[1].split())
    nbr, _, _ = po.build_neighbors(pos, 64, 6.0)
    ref, _ = po.attn_fwd(po.AttnProblem(L=2, H=8, value_mode=po.VALUE_DENSE), q, k, v, pos, nbr)
    assert abs(s - ref.sum()) <= 1e-5 * np.abs(ref).sum()
    assert abs(s2 - (ref ** 2).sum()) <= 1e-5 * (ref ** 2).sum()
