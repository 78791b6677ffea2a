"""Generate tests/golden/so3_ref.npz from the REFERENCE's own so3 headers
(compiled in place by oracle/build_ref.sh through the Eigen shim).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The GPU box has no /root/reference, so the parity tests read these
committed vectors instead.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402


def main():
    po.build()
    R = po.ref()
    rng = np.random.default_rng(20260117)
    pts = rng.standard_normal((64, 3)) * rng.uniform(0.2, 6.0, (64, 1))
    out = {"points": pts}
    for l in range(5):
        Y = np.zeros((64, 2 * l + 1))
        for i, p in enumerate(pts):
            R.esref_solid_harmonics(l, po._p(po._c(p)), po._p(Y[i]))
        out[f"solid_l{l}"] = Y
    for l1 in range(5):
        for l2 in range(5):
            for lo in range(abs(l1 - l2), min(l1 + l2, 4) + 1):
                b = np.zeros((2 * lo + 1) * (2 * l1 + 1) * (2 * l2 + 1))
                R.esref_cg_real(l1, l2, lo, po._p(b))
                out[f"cg_{l1}{l2}{lo}"] = b.reshape(2 * lo + 1, 2 * l1 + 1, 2 * l2 + 1)
    # dense tensor products of random blocks (tensor_product.hpp:18)
    for (l1, l2, lo) in [(1, 1, 0), (1, 1, 1), (1, 1, 2), (2, 1, 3), (2, 2, 2), (4, 2, 3), (4, 4, 4)]:
        u = rng.standard_normal((2 * l1 + 1, 5))
        v = rng.standard_normal((2 * l2 + 1, 5))
        o = np.zeros((2 * lo + 1, 5))
        R.esref_tensor_product_dense(po._p(po._c(u)), l1, 5, po._p(po._c(v)), l2, 5, lo, po._p(o))
        out[f"tp_{l1}{l2}{lo}_u"], out[f"tp_{l1}{l2}{lo}_v"], out[f"tp_{l1}{l2}{lo}_out"] = u, v, o
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "so3_ref.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays")


if __name__ == "__main__":
    main()
