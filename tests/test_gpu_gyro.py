"""GPU: the gyro-permutation search (§8(f) row 1) against the reference's own runs
(tests/golden/gyro.npz + gyro_reports.json, generator tests/golden/make_golden_gyro.py):
identical sigma_o, sigma_i, both masks and the whole PruneReport (every retention log entry
bit-equal) for OCP + ICP runs, the ablation variants and a tie-heavy matrix; plus the ICP cost
kernel against the reference's double loop."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import permutation as P  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "gyro_reports.json")) as fh:
    REPORTS = json.load(fh)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "gyro.npz"))


@pytest.mark.parametrize("name", sorted(REPORTS))
def test_gyro_permute_matches_reference(g, name):
    m, n, V, N, M, sv, oi, ii, seed, ocs, ics = REPORTS[name]["cfg"]
    cfg = H.HiNMConfig(vector_size=V, nm_keep=N, nm_group=M, vector_sparsity=sv,
                       ocp_max_iters=oi, icp_max_iters=ii, seed=seed)
    sigma, masks, rep = P.gyro_permute(g[f"{name}_W"], cfg, ocp_strategy=ocs, icp_strategy=ics)
    assert np.array_equal(sigma.sigma_o, g[f"{name}_sigma_o"])
    lens = g[f"{name}_sigma_i_len"]
    assert [len(o) for o in sigma.sigma_i] == lens.tolist()
    assert np.array_equal(np.concatenate(sigma.sigma_i), g[f"{name}_sigma_i"])
    assert np.array_equal(masks.vector_mask, g[f"{name}_vmask"])
    assert np.array_equal(masks.element_mask, g[f"{name}_emask"])
    assert rep.to_dict() == REPORTS[name]["report"]


def test_balanced_kmeans_matches_reference(g):
    """k-means++ seeding + capacitated Lloyd rounds with the distances on the GPU (hinm_sq_dists,
    numpy pairwise order): the reference's labels bit-for-bit."""
    for t in range(6):
        k = t + 2
        pts = g[f"km_pts{t}"]
        groups = P.balanced_kmeans(pts, k, 6, np.random.default_rng(t))
        lab = np.empty(pts.shape[0], dtype=np.int64)
        for c, idx in enumerate(groups):
            lab[idx] = c
        assert np.array_equal(lab, g[f"km_lab{t}"]), t


def test_sq_dists_bit_exact_with_numpy():
    rng = np.random.default_rng(4)
    for P_, C, F in ((37, 5, 1), (64, 7, 3), (50, 9, 129), (33, 4, 4096), (12, 3, 11008)):
        pts = rng.standard_normal((P_, F)) * rng.choice([1.0, 1e-3, 1e3], size=(P_, F))
        cents = rng.standard_normal((C, F))
        ref = ((pts[:, None, :] - cents[None, :, :]) ** 2).sum(axis=-1)
        assert np.array_equal(P._Dists(pts)(cents), ref), (P_, C, F)
        assert np.array_equal(P._Dists(pts)(cents[0])[:, 0], ((pts - cents[0]) ** 2).sum(axis=1))


def _ref_icp_costs(vals, rem, samp, N):
    G = len(samp)
    C = np.empty((G, G))
    for i in range(G):
        base = vals[:, rem[i]]
        bt = float(base.sum())
        for j in range(G):
            union = np.concatenate([base, vals[:, [samp[j]]]], axis=1)
            kept = float(np.sort(union, axis=1)[:, -N:].sum())
            C[i, j] = bt + float(vals[:, samp[j]].sum()) - kept
    return C


@pytest.mark.parametrize("V,M,N", [(64, 4, 2), (128, 4, 2), (16, 4, 1), (8, 8, 3)])
def test_icp_cost_kernel_bit_exact(V, M, N):
    rng = np.random.default_rng(V + M + N)
    tile = np.abs(rng.standard_normal((V, 96))) * rng.choice([1.0, 1e-3, 1e2], size=(V, 96))
    surv = np.sort(rng.permutation(96)[:M * 10])
    vals = tile[:, surv]
    G = 10
    groups = [list(range(q * M, (q + 1) * M)) for q in range(G)]
    picks = [int(rng.integers(M)) for _ in groups]
    samp = [grp[p] for grp, p in zip(groups, picks)]
    rem = [[x for q, x in enumerate(grp) if q != p] for grp, p in zip(groups, picks)]
    ref = _ref_icp_costs(vals, rem, samp, N)
    got = P._IcpCostsGPU(vals, M, N)(np.array(rem), np.array(samp))
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("m,n,V,sv,samples", [(256, 128, 64, 0.5, 8), (512, 96, 32, 0.75, 4),
                                              (384, 4096, 64, 0.5, 16), (128, 11008, 64, 0.5, 16)])
def test_ocp_cost_kernel_matches_reference_loop(m, n, V, sv, samples):
    """hinm_ocp_costs (one CTA per pair, sort + merge) vs the reference's per-pair lexsort +
    np.partition (permutation.py:295-327): the same retained multiset, so equal up to floating-point
    association (relative 1e-12); the assignment picked from either matrix is identical."""
    rng = np.random.default_rng(m + n)
    scores = np.abs(rng.standard_normal((m, n)))
    scores[:, : n // 8] *= 1e-3                       # spread of magnitudes, as in real saliency
    vcfg = H.validate_config(H.HiNMConfig(V, 2, 4, sv), (m, n))
    tiles = P._tiles_of(rng.permutation(m), V)
    rems, samp = P.sample_channels(tiles, samples, rng)
    pool = np.concatenate(samp)
    clusters = [np.sort(pool[q]) for q in P.balanced_kmeans(scores[pool], len(tiles), samples, rng)]
    host = P._ocp_costs_host(scores, rems, clusters, vcfg)
    dev = P._ocp_costs(scores, rems, clusters, vcfg)
    np.testing.assert_allclose(dev, host, rtol=1e-12, atol=1e-9)
    assert np.array_equal(P.hungarian(dev), P.hungarian(host))
