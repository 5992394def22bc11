"""Pin the CPU oracle against golden vectors produced by the real reference.

The oracle (oracle/hinm_oracle.py) is the checker for every GPU parity test, so
it must itself reproduce the reference bit-for-bit on the reference's own KATs,
its round-trip instances and ~60 random/tie-heavy/empty-tile instances.
"""

import json
import os

import numpy as np
import pytest

import hinm_oracle as O
from conftest import GOLDEN, case, load_small
from paper_2407_20496_b200 import synth

Z, NAMES = load_small()


@pytest.mark.parametrize("key", NAMES)
def test_oracle_matches_reference_case(key):
    d = case(Z, key)
    m, n, V, N, M = d["m"], d["n"], d["V"], d["N"], d["M"]
    S = np.abs(d["W"])
    vm, counts, _ = O.vector_prune(S, d["sigma_o"], V, M, d["total_keep"])
    assert np.array_equal(vm, d["vector_mask"])
    # sigma_i stored in the case is what the reference used (gyro / ascending / permuted)
    surv = O.survivors(vm)
    for t in range(m // V):
        assert set(surv[t].tolist()) == set(d["sigma_i"][t].tolist())
    em, pos = O.nm_prune(S, d["sigma_o"], d["sigma_i"], V, N, M)
    assert np.array_equal(em, d["element_mask"])
    tiles = O.encode(d["W"], d["sigma_o"], d["sigma_i"], pos, V, N, M)
    vidx = np.concatenate([t[0] for t in tiles])
    nmi = np.concatenate([t[1].ravel() for t in tiles])
    kv = np.concatenate([t[2].ravel() for t in tiles])
    assert np.array_equal(vidx, d["vector_index"])
    assert np.array_equal(nmi, d["nm_index"])
    assert np.array_equal(kv, d["kept_values"])  # bit-exact copies of weights
    assert np.array_equal(O.decode(tiles, (m, n), V, N, M), d["decode"])
    if "X" in d:
        Y = O.hinm_spmm(tiles, d["X"], m, V, N, M)
        assert O.relative_error(Y, d["Y"]) <= 1e-12


def test_greedy_equals_sorted_allocation():
    """The vectorised budget (global sort of (-gain, q, t)) equals the reference greedy loop."""
    rng = np.random.default_rng(5)
    for trial in range(200):
        T = int(rng.integers(1, 9))
        G = int(rng.integers(1, 12))
        if trial % 2:
            g = rng.integers(0, 4, size=(T, G)).astype(float)   # tie-heavy
        else:
            g = rng.random((T, G))
        g = -np.sort(-g, axis=1)                                 # non-increasing per tile
        k = int(rng.integers(0, T * G + 1))
        assert np.array_equal(O.allocate_budget_greedy(g, k), O.allocate_budget_sorted(g, k))


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 64, 127, 128, 129, 300):
        for _ in range(20):
            a = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, size=n)
            assert O.pairwise_sum(a) == a.reshape(1, n).sum(axis=1)[0]


def test_cfg1_gyro_fixture():
    """cfg1 768x3072 with the reference gyro sigma (OCP, icp_max_iters=0): oracle == reference."""
    z = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    W = synth.randn_bf16((768, 3072), 0).astype(np.float64)
    so = z["sigma_o"].astype(np.int64)
    ptr = z["sigma_i_ptr"]
    si = [z["sigma_i"][ptr[t]:ptr[t + 1]].astype(np.int64) for t in range(12)]
    r = O.compress(W, so, 64, 2, 4, 12 * 1536, sigma_i=si)
    assert np.array_equal(np.packbits(r["vector_mask"], axis=1), z["vector_mask"])
    vidx = np.concatenate([t[0] for t in r["tiles"]])
    nmi = np.concatenate([t[1].ravel() for t in r["tiles"]])
    assert np.array_equal(vidx, z["vector_index"].astype(np.int64))
    assert np.array_equal(nmi, z["nm_index"])
    X = synth.randn_bf16((3072, 512), 1).astype(np.float64)
    Y = O.hinm_spmm(r["tiles"], X, 768, 64, 2, 4)
    assert O.relative_error(Y, z["Y"].astype(np.float64)) < 1e-6


@pytest.mark.parametrize("name", ["llama_down", "llama_up"])
def test_large_digests(name):
    """LLaMA-7B FFN shapes: oracle encoding digests equal the reference's."""
    import hashlib

    spec = json.load(open(os.path.join(GOLDEN, "large.json")))[name]
    m, n = spec["m"], spec["n"]
    W = synth.randn_bf16((m, n), spec["w_seed"]).astype(np.float64)
    so = synth.random_sigma_o(m, spec["sigma_o_seed"])
    vm, counts, _ = O.vector_prune(np.abs(W), so, 64, 4, (m // 64) * (n // 2))
    assert counts.tolist() == spec["counts"]
    si = synth.permute_survivors(O.survivors(vm), spec["sigma_i_seed"])
    em, pos = O.nm_prune(np.abs(W), so, si, 64, 2, 4)
    tiles = O.encode(W, so, si, pos, 64, 2, 4)
    vidx = np.concatenate([t[0] for t in tiles]).astype("<i4")
    nmi = np.concatenate([t[1].ravel() for t in tiles]).astype(np.uint8)
    assert hashlib.sha256(vidx.tobytes()).hexdigest() == spec["vector_index_int32_sha256"]
    assert hashlib.sha256(nmi.tobytes()).hexdigest() == spec["nm_index_u8_sha256"]
    assert hashlib.sha256(np.ascontiguousarray(em).tobytes()).hexdigest() == spec["element_mask_sha256"]
