"""Run the bf16 parity tests again with the tcgen05 attention kernel enabled
(ES_ATTN_TC=1 is read once per process, hence the subprocess), so a plain
`pytest -m gpu` covers both attention forward kernels."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tensor_core_attention_parity():
    env = dict(os.environ, ES_ATTN_TC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
                        "bf16 or tensor_core or row_sharded"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
