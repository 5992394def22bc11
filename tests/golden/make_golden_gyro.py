"""Golden vectors for the gyro-permutation search (§8(f) row 1), produced by the REAL reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_gyro.py

Writes tests/golden/gyro.npz (+ gyro_reports.json):
  hungarian : 60 cost matrices (real, small-integer / tie-heavy, duplicate columns) and the
              reference's lexicographic optimal assignments
  kmeans    : balanced_kmeans(features, k, size, default_rng(s)) cluster labels
  gyro_<i>  : gyro_permute(W, cfg[, strategies]) -> sigma_o, sigma_i, masks, report, for small
              and medium instances (OCP + ICP, ablations, a tie-heavy matrix)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import hinm  # noqa: E402  (the reference)
from hinm.permutation import balanced_kmeans, hungarian  # noqa: E402

from paper_2407_20496_b200 import synth  # noqa: E402

CASES = [
    # (name, m, n, V, N, M, s_v, ocp_iters, icp_iters, seed, ocp_strategy, icp_strategy, weights)
    ("small_full", 64, 128, 16, 2, 4, 0.5, 3, 4, 0, "sampled", "hungarian", "randn"),
    ("small_seed1", 64, 128, 16, 2, 4, 0.5, 2, 3, 1, "sampled", "hungarian", "randn"),
    ("v8_14", 32, 64, 8, 1, 4, 0.25, 2, 3, 2, "sampled", "hungarian", "randn"),
    ("ties", 32, 64, 8, 2, 4, 0.5, 2, 3, 3, "sampled", "hungarian", "ties"),
    ("kmeans_all", 64, 64, 16, 2, 4, 0.5, 0, 3, 4, "kmeans_all", "hungarian", "randn"),
    ("swap", 32, 32, 8, 2, 4, 0.5, 1, 2, 5, "sampled", "swap", "randn"),
    ("icp_only", 128, 256, 64, 2, 4, 0.5, 0, 3, 6, "identity", "hungarian", "randn"),
    ("medium", 256, 512, 64, 2, 4, 0.5, 2, 2, 7, "sampled", "hungarian", "randn"),
]


def main():
    out, reports = {}, {}
    rng = np.random.default_rng(2024)
    mats = []
    for t in range(60):
        n = int(rng.integers(1, 40))
        kind = t % 3
        if kind == 0:
            C = rng.random((n, n)) * 100
        elif kind == 1:
            C = rng.integers(0, 3, (n, n)).astype(float)
        else:
            C = rng.random((n, n))
            C[:, rng.integers(0, n, n)] = C[:, :1]
        out[f"hung_C{t}"] = C
        out[f"hung_a{t}"] = hungarian(C)
    for t in range(6):
        k = t + 2
        pts = rng.standard_normal((6 * k, 3))
        labels = np.empty(pts.shape[0], dtype=np.int64)
        for c, idx in enumerate(balanced_kmeans(pts, k, 6, np.random.default_rng(t))):
            labels[idx] = c
        out[f"km_pts{t}"] = pts
        out[f"km_lab{t}"] = labels
    for i, (name, m, n, V, N, M, sv, oi, ii, seed, ocs, ics, wk) in enumerate(CASES):
        W = (synth.randn_bf16((m, n), 100 + i) if wk == "randn"
             else synth.tie_heavy_bf16((m, n), 100 + i)).astype(np.float64)
        cfg = hinm.HiNMConfig(vector_size=V, nm_keep=N, nm_group=M, vector_sparsity=sv,
                              ocp_max_iters=oi, icp_max_iters=ii, seed=seed)
        sigma, masks, rep = hinm.gyro_permute(W, cfg, ocp_strategy=ocs, icp_strategy=ics)
        out[f"{name}_W"] = W
        out[f"{name}_sigma_o"] = np.asarray(sigma.sigma_o, dtype=np.int64)
        out[f"{name}_sigma_i"] = np.concatenate([np.asarray(o, dtype=np.int64) for o in sigma.sigma_i])
        out[f"{name}_sigma_i_len"] = np.array([len(o) for o in sigma.sigma_i], dtype=np.int64)
        out[f"{name}_vmask"] = masks.vector_mask
        out[f"{name}_emask"] = masks.element_mask
        reports[name] = {"cfg": [m, n, V, N, M, sv, oi, ii, seed, ocs, ics], "report": rep.to_dict()}
        print(name, "fallback", rep.fallback_used, "retained", rep.retained_saliency)
    np.savez_compressed(os.path.join(HERE, "gyro.npz"), **out)
    with open(os.path.join(HERE, "gyro_reports.json"), "w") as fh:
        json.dump(reports, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
