"""Gyro-permutation search, host parts (no GPU): the native lexicographic assignment against the
reference's outputs (tests/golden/gyro.npz, generator tests/golden/make_golden_gyro.py); the
balanced k-means (GPU distances) is checked in test_gpu_gyro.py."""

import os

import numpy as np
import pytest

from paper_2407_20496_b200 import permutation as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "gyro.npz"))


def test_hungarian_matches_reference(g):
    n_cases = sum(1 for k in g.files if k.startswith("hung_C"))
    assert n_cases == 60
    for t in range(n_cases):
        assert np.array_equal(P.hungarian(g[f"hung_C{t}"]), g[f"hung_a{t}"]), t


def test_hungarian_argument_checks():
    with pytest.raises(ValueError):
        P.hungarian(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        P.hungarian(np.array([[0.0, np.inf], [1.0, 2.0]]))
    assert P.hungarian(np.zeros((0, 0))).size == 0


def test_hungarian_is_optimal_and_lexicographic():
    rng = np.random.default_rng(3)
    C = rng.integers(0, 2, (30, 30)).astype(float)
    a = P.hungarian(C)
    assert sorted(a.tolist()) == list(range(30))
    from itertools import permutations  # brute force on a tiny one
    D = rng.integers(0, 3, (6, 6)).astype(float)
    best = min(permutations(range(6)), key=lambda p: (sum(D[i, p[i]] for i in range(6)), p))
    assert tuple(P.hungarian(D)) == best


def test_sample_channels_sizes():
    parts = [P.Partition("output", np.arange(i * 8, i * 8 + 8), 8) for i in range(3)]
    rems, samples = P.sample_channels(parts, 3, np.random.default_rng(0))
    assert all(r.members.size == 5 and s.size == 3 for r, s in zip(rems, samples))
    for r, s, p in zip(rems, samples, parts):
        assert sorted(np.concatenate([r.members, s]).tolist()) == p.members.tolist()
