import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The parity systems are small (< 74 query tiles), where the library would
# pick the SIMT attention forward; force the tcgen05 kernel wherever its shape
# is supported so the tests cover it (tests/test_gpu_tc_path.py re-runs the
# bf16 cases with ES_ATTN_TC=0 for the SIMT kernel).
os.environ.setdefault("ES_ATTN_TC", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: larger parity sizes")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    pyoracle.build()
    return pyoracle


@pytest.fixture(scope="session")
def ref(oracle):
    if not oracle.ref_available():
        pytest.skip("reference-built oracle/_ref/libesref.so not available (needs /root/reference to build)")
    return oracle.ref()


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(params=["tc_kv", "simt_dk", "tc_dk"])
def dk_path(request, monkeypatch):
    """The backward variants of a molecule batch: the tensor-core key pass
    (default: dv + dscores, then dk and dq on the tensor cores), the SIMT key
    pass with dk (ES_KV_TC=0), and the SIMT key pass without dk followed by the
    tensor-core dk pass (ES_KV_TC=0, ES_DK_TC=1)."""
    monkeypatch.setenv("ES_KV_TC", "1" if request.param == "tc_kv" else "0")
    monkeypatch.setenv("ES_DK_TC", "1" if request.param == "tc_dk" else "0")
    return request.param
