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
