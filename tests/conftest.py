"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with ``-m gpu``).
The oracle under ``oracle/`` is test infrastructure: tests import it as the checker.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_small():
    z = np.load(os.path.join(GOLDEN, "small.npz"))
    names = [str(s) for s in z["names"]]
    return z, names


def case(z, key):
    """Unpack one golden case into plain python/numpy values."""
    meta = z[key + "meta"]
    m, n, V, N, M, num, den = (int(x) for x in meta)
    ptr = z[key + "sigma_i_ptr"]
    sig = z[key + "sigma_i"]
    tptr = z[key + "tile_ptr"]
    d = dict(m=m, n=n, V=V, N=N, M=M, s_v=(num, den), W=z[key + "W"], sigma_o=z[key + "sigma_o"],
             sigma_i=[sig[ptr[t]:ptr[t + 1]] for t in range(len(ptr) - 1)],
             vector_mask=z[key + "vector_mask"], element_mask=z[key + "element_mask"],
             vector_index=z[key + "vector_index"], tile_ptr=tptr, nm_index=z[key + "nm_index"],
             kept_values=z[key + "kept_values"], decode=z[key + "decode"])
    T = m // V
    d["total_keep"] = T * (n * (den - num) // den)
    if key + "X" in z.files:
        d["X"] = z[key + "X"]
        d["Y"] = z[key + "Y"]
    return d


@pytest.fixture(scope="session")
def golden_small():
    return load_small()
