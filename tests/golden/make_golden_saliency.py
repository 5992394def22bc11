"""Golden vectors for the external-saliency path, produced by the REAL reference (build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_saliency.py

The reference's `encode --saliency` chain (cli.py:63-69 load_saliency, cli.py:185-194) feeds an
external score matrix S to vector_prune / nm_prune and takes the kept values from W.  Library calls
accept any real-valued S (as_values, no sign check), so the cases include negative and tie-heavy
scores.  Writes tests/golden/saliency.npz: the reference's outputs (vector_mask, element_mask,
vector_index, nm_index, kept_values, tile_ptr, Y = hinm_spmm(enc, X)); the inputs are regenerated
by `inputs()` (pure numpy, seeded -- tests/test_gpu_image.py carries the same generator).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import hinm  # noqa: E402  (the reference)
from hinm.pruning import survivors_per_tile  # noqa: E402

from paper_2407_20496_b200 import synth  # noqa: E402

# name, m, n, V, s_v, score kind, seed
CASES = [
    ("pos64", 256, 512, 64, 0.5, "abs_normal", 1),
    ("neg32", 256, 512, 32, 0.5, "normal", 2),
    ("neg128", 384, 768, 128, 0.5, "normal_f32", 3),
    ("ties64", 128, 256, 64, 0.5, "int", 4),
    ("keep25_64", 256, 1024, 64, 0.75, "normal", 5),
]


def scores(kind, shape, seed):
    rng = np.random.default_rng(1000 + seed)
    if kind == "abs_normal":
        return np.abs(rng.standard_normal(shape))
    if kind == "normal":
        return rng.standard_normal(shape)
    if kind == "normal_f32":
        return rng.standard_normal(shape).astype(np.float32).astype(np.float64)
    return rng.integers(-3, 4, size=shape).astype(np.float64)


def inputs(m, n, kind, seed):
    """W, S, sigma_o, X of a case (sigma_i = ascending survivors permuted by seed 10*seed + 2)."""
    return (synth.randn_bf16((m, n), 10 * seed).astype(np.float64), scores(kind, (m, n), seed),
            synth.random_sigma_o(m, 10 * seed + 1), synth.randn_bf16((n, 24), 10 * seed + 3).astype(np.float64))


def main():
    out = {}
    for name, m, n, V, sv, kind, seed in CASES:
        W, S, so, X = inputs(m, n, kind, seed)
        cfg = hinm.HiNMConfig(vector_size=V, nm_keep=2, nm_group=4, vector_sparsity=sv)
        vm = hinm.vector_prune(S, cfg, so)
        si = synth.permute_survivors(survivors_per_tile(vm), 10 * seed + 2)
        sigma = hinm.GyroPermutation(so, tuple(si))
        em = hinm.nm_prune(S, vm, cfg, sigma)
        enc = hinm.encode(W, hinm.MaskPair(vm, em), sigma, cfg)
        p = name + "_"
        out[p + "vector_mask"], out[p + "element_mask"] = vm, em
        out[p + "vector_index"] = np.concatenate([t.vector_index for t in enc.tiles])
        out[p + "nm_index"] = np.concatenate([t.nm_index.ravel() for t in enc.tiles]).astype(np.uint8)
        out[p + "kept_values"] = np.concatenate([t.kept_values.ravel() for t in enc.tiles])
        out[p + "tile_ptr"] = np.concatenate([[0], np.cumsum([t.vector_index.size for t in enc.tiles])])
        out[p + "Y"] = hinm.hinm_spmm(enc, X)
        print(name, "k_t:", np.diff(out[p + "tile_ptr"]).tolist()[:6], "...")
    out["names"] = np.array([c[0] for c in CASES])
    out["cases"] = np.array([[m, n, V, int(sv * 100), seed] for _, m, n, V, sv, _, seed in CASES])
    out["kinds"] = np.array([c[5] for c in CASES])
    np.savez_compressed(os.path.join(HERE, "saliency.npz"), **out)


if __name__ == "__main__":
    main()
