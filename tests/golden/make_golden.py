"""Generate golden vectors by running the REAL reference package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes (committed, small):
  tests/golden/small.npz        -- KATs from the reference test-suite plus ~60 random
                                   instances (general V, N:M, s_v, ties, empty tiles)
  tests/golden/cfg1.npz         -- 768x3072, V=64, 2:4, s_v=0.5, gyro sigma (OCP only,
                                   icp_max_iters=0) + hinm_spmm at B=512
  tests/golden/large.json       -- LLaMA-7B FFN shapes: SHA-256 digests of the reference
                                   encoding + per-tile counts; Y for B=16 in large_y.npz

Every array stored here is an OUTPUT of the reference functions
(``vector_prune``/``nm_prune``/``encode``/``decode``/``hinm_spmm``); inputs are
regenerated deterministically from ``paper_2407_20496_b200.synth``.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import hinm  # noqa: E402  (the reference)
from hinm.pruning import survivors_per_tile  # noqa: E402

from paper_2407_20496_b200 import synth  # noqa: E402


def ragged(arrs, dtype):
    arrs = [np.asarray(a, dtype=dtype).ravel() for a in arrs]
    ptr = np.zeros(len(arrs) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([a.size for a in arrs])
    flat = np.concatenate(arrs) if arrs else np.empty(0, dtype)
    return flat, ptr


def run_reference(W, cfg, sigma_o, sigma_i_mode, X, seed):
    """vector_prune -> (sigma_i) -> nm_prune -> encode -> decode / hinm_spmm with the reference."""
    S = hinm.magnitude_saliency(W)
    vm = hinm.vector_prune(S, cfg, sigma_o)
    surv = survivors_per_tile(vm)
    if sigma_i_mode == "ascending":
        sig_i = surv
    else:
        sig_i = synth.permute_survivors(surv, seed)
    sigma = hinm.GyroPermutation(np.asarray(sigma_o), tuple(sig_i))
    em = hinm.nm_prune(S, vm, cfg, sigma)
    masks = hinm.MaskPair(vm, em)
    enc = hinm.encode(W, masks, sigma, cfg)
    m, n = W.shape
    dec = hinm.decode(enc, (m, n))
    Y = hinm.hinm_spmm(enc, X) if X is not None else None
    return vm, em, sigma, enc, dec, Y


def pack_case(store, key, W, cfg, sigma_o, sigma, vm, em, enc, dec, X, Y):
    vidx, vptr = ragged([t.vector_index for t in enc.tiles], np.int64)
    nmi, _ = ragged([t.nm_index for t in enc.tiles], np.uint8)
    kv, _ = ragged([t.kept_values for t in enc.tiles], np.float64)
    sig_i, sptr = ragged(sigma.sigma_i, np.int64)
    s_v = Fraction(cfg.vector_sparsity).limit_denominator(10**6) if not isinstance(
        cfg.vector_sparsity, Fraction) else cfg.vector_sparsity
    store[key + "meta"] = np.array(
        [W.shape[0], W.shape[1], cfg.vector_size, cfg.nm_keep, cfg.nm_group,
         s_v.numerator, s_v.denominator], dtype=np.int64)
    store[key + "W"] = np.asarray(W, dtype=np.float64)
    store[key + "sigma_o"] = np.asarray(sigma_o, dtype=np.int64)
    store[key + "sigma_i"] = sig_i
    store[key + "sigma_i_ptr"] = sptr
    store[key + "vector_mask"] = vm
    store[key + "element_mask"] = em
    store[key + "vector_index"] = vidx
    store[key + "tile_ptr"] = vptr
    store[key + "nm_index"] = nmi
    store[key + "kept_values"] = kv
    store[key + "decode"] = dec
    if X is not None:
        store[key + "X"] = np.asarray(X, dtype=np.float64)
        store[key + "Y"] = Y


def small_cases():
    store = {}
    names = []
    # (1) the reference test-suite's own round-trip instances (test_pruning.py:226-237):
    #     gyro_permute on N(0,1) 8x16, V=4, 2:4, s_v=0.5, seed 3, rng 1234
    rng = np.random.default_rng(1234)
    cfg = hinm.HiNMConfig(vector_size=4, nm_keep=2, nm_group=4, vector_sparsity=0.5, seed=3)
    for i in range(20):
        W = rng.normal(size=(8, 16))
        sigma, masks, _ = hinm.gyro_permute(W, cfg)
        enc = hinm.encode(W, masks, sigma, cfg)
        dec = hinm.decode(enc, (8, 16))
        X = synth.randn_bf16((16, 8), 500 + i).astype(np.float64)
        Y = hinm.hinm_spmm(enc, X)
        key = f"gyro{i}_"
        pack_case(store, key, W, cfg, sigma.sigma_o, sigma, masks.vector_mask,
                  masks.element_mask, enc, dec, X, Y)
        names.append(key)

    # (2) KATs of test_pruning.py / conftest.py
    kats = []
    S = np.array([[9.0, 9.0], [1.0, 1.0], [9.0, 9.0], [1.0, 1.0]])  # conftest.py:12-26
    kats.append(("kat_ocp_", S, hinm.HiNMConfig(2, 1, 1, 0.5), np.array([0, 2, 1, 3])))
    kats.append(("kat_uniform_", np.ones((4, 8)), hinm.HiNMConfig(2, 1, 2, 0.5), np.arange(4)))
    kats.append(("kat_keepall_", np.ones((4, 4)), hinm.HiNMConfig(2, 1, 2, 0.0), np.arange(4)))
    rng2 = np.random.default_rng(1234)
    kats.append(("kat_sortoracle_", np.abs(rng2.normal(size=(4, 16))),
                 hinm.HiNMConfig(4, 1, 2, 0.5), np.arange(4)))
    kats.append(("kat_top2_", np.array([[1.0, 2.0, 3.0, 4.0]]), hinm.HiNMConfig(1, 2, 4, 0.0),
                 np.array([0])))
    kats.append(("kat_tie_", np.array([[5.0, 5.0, 5.0, 5.0]]), hinm.HiNMConfig(1, 2, 4, 0.0),
                 np.array([0])))
    kats.append(("kat_icp_", np.tile([9.0, 8.0, 7.0, 6.0, 1.0, 1.0, 1.0, 1.0], (2, 1)),
                 hinm.HiNMConfig(2, 2, 4, 0.0), np.arange(2)))
    for key, W, cfg, so in kats:
        vm, em, sigma, enc, dec, _ = run_reference(W, cfg, so, "ascending", None, 0)
        pack_case(store, key, W, cfg, so, sigma, vm, em, enc, dec, None, None)
        names.append(key)
    # sigma_i-driven grouping KAT (test_pruning.py:137-146)
    W = np.array([[9.0, 8.0, 7.0, 6.0, 1.0, 1.0, 1.0, 1.0]])
    cfg = hinm.HiNMConfig(1, 2, 4, 0.0)
    sigma = hinm.GyroPermutation(np.array([0]), (np.array([0, 3, 4, 5, 1, 2, 6, 7]),))
    vm = np.ones((1, 8), bool)
    em = hinm.nm_prune(W, vm, cfg, sigma)
    enc = hinm.encode(W, hinm.MaskPair(vm, em), sigma, cfg)
    pack_case(store, "kat_sigmai_", W, cfg, np.array([0]), sigma, vm, em, enc,
              hinm.decode(enc, W.shape), None, None)
    names.append("kat_sigmai_")

    # (3) random bf16 instances over the config space, random sigma_o / sigma_i, B=16
    specs = []
    for V in (1, 2, 4, 8, 16, 32, 64):
        for (N, M) in ((1, 1), (1, 2), (2, 4), (1, 4), (2, 8), (3, 8)):
            for s_v in (0.0, 0.25, 0.5, 0.75):
                specs.append((V, N, M, s_v))
    prng = np.random.default_rng(77)
    chosen = [specs[i] for i in prng.choice(len(specs), size=48, replace=False)]
    chosen += [(64, 2, 4, 0.5), (32, 2, 4, 0.5), (128, 2, 4, 0.5), (64, 2, 4, 0.75),
               (64, 2, 4, 0.0), (16, 2, 4, 0.5)]
    for ci, (V, N, M, s_v) in enumerate(chosen):
        T = int(prng.integers(1, 5))
        m = V * T
        # smallest n with n*(1-s_v) a multiple of M, scaled
        base = next(k for k in range(1, 64) if (Fraction(k) * (1 - Fraction(s_v))).denominator == 1
                    and int(Fraction(k) * (1 - Fraction(s_v))) % M == 0
                    and int(Fraction(k) * (1 - Fraction(s_v))) > 0)
        n = base * int(prng.integers(1, max(2, 96 // base)))
        cfg = hinm.HiNMConfig(V, N, M, s_v)
        kind = ci % 3
        if kind == 0:
            W = synth.randn_bf16((m, n), 1000 + ci)
        elif kind == 1:
            W = synth.tie_heavy_bf16((m, n), 1000 + ci)
        else:  # one starved tile -> possibly empty (global budget)
            W = synth.randn_bf16((m, n), 1000 + ci)
            W[:V] = synth.bf16_round(W[:V] * np.float32(1e-3))
        so = synth.random_sigma_o(m, 2000 + ci)
        mode = "ascending" if ci % 2 == 0 else "permuted"
        X = synth.randn_bf16((n, 16), 3000 + ci).astype(np.float64)
        vm, em, sigma, enc, dec, Y = run_reference(W.astype(np.float64), cfg, so, mode, X,
                                                   4000 + ci)
        key = f"rand{ci}_"
        pack_case(store, key, W.astype(np.float64), cfg, so, sigma, vm, em, enc, dec, X, Y)
        names.append(key)
    # n == 1 column (numpy pairwise axis-0 path)
    W = synth.randn_bf16((24, 1), 99).astype(np.float64)
    cfg = hinm.HiNMConfig(8, 1, 1, 0.0)
    so = synth.random_sigma_o(24, 98)
    vm, em, sigma, enc, dec, _ = run_reference(W, cfg, so, "ascending", None, 0)
    pack_case(store, "ncol1_", W, cfg, so, sigma, vm, em, enc, dec, None, None)
    names.append("ncol1_")
    store["names"] = np.array(names)
    return store


def cfg1_case():
    m, n, B = 768, 3072, 512
    W = synth.randn_bf16((m, n), 0).astype(np.float64)
    X = synth.randn_bf16((n, B), 1).astype(np.float64)
    cfg = hinm.HiNMConfig(vector_size=64, nm_keep=2, nm_group=4, vector_sparsity=0.5,
                          seed=0, icp_max_iters=0)
    t0 = time.time()
    sigma, masks, report = hinm.gyro_permute(W, cfg)
    t_gyro = time.time() - t0
    t0 = time.time()
    enc = hinm.encode(W, masks, sigma, cfg)
    Y = hinm.hinm_spmm(enc, X)
    t_spmm = time.time() - t0
    vidx, vptr = ragged([t.vector_index for t in enc.tiles], np.int64)
    nmi, _ = ragged([t.nm_index for t in enc.tiles], np.uint8)
    sig_i, sptr = ragged(sigma.sigma_i, np.int64)
    print(f"cfg1: gyro {t_gyro:.1f}s, encode+spmm {t_spmm:.1f}s")
    return {
        "sigma_o": sigma.sigma_o.astype(np.int16), "sigma_i": sig_i.astype(np.int16),
        "sigma_i_ptr": sptr, "vector_index": vidx.astype(np.int16), "tile_ptr": vptr,
        "nm_index": nmi, "Y": Y.astype(np.float32),
        "vector_mask": np.packbits(masks.vector_mask, axis=1),
        "element_mask_digest": np.frombuffer(hashlib.sha256(
            np.ascontiguousarray(masks.element_mask).tobytes()).digest(), np.uint8),
    }


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def large_cases():
    out, ys = {}, {}
    for name, (m, n) in {"llama_down": (4096, 11008), "llama_up": (11008, 4096)}.items():
        W = synth.randn_bf16((m, n), 0).astype(np.float64)
        so = synth.random_sigma_o(m, 2)
        cfg = hinm.HiNMConfig(vector_size=64, nm_keep=2, nm_group=4, vector_sparsity=0.5)
        X = synth.randn_bf16((n, 16), 1).astype(np.float64)
        t0 = time.time()
        vm, em, sigma, enc, dec, Y = run_reference(W, cfg, so, "permuted", X, 3)
        dt = time.time() - t0
        vidx, vptr = ragged([t.vector_index for t in enc.tiles], np.int64)
        nmi, _ = ragged([t.nm_index for t in enc.tiles], np.uint8)
        counts = np.diff(vptr)
        out[name] = {
            "m": m, "n": n, "V": 64, "N": 2, "M": 4, "s_v": "1/2",
            "w_seed": 0, "sigma_o_seed": 2, "sigma_i_seed": 3, "x_seed": 1, "B": 16,
            "counts": counts.tolist(),
            "vector_index_int32_sha256": digest(vidx.astype("<i4")),
            "nm_index_u8_sha256": digest(nmi.astype(np.uint8)),
            "element_mask_sha256": digest(em),
            "reference_seconds": round(dt, 2),
        }
        ys[name] = Y.astype(np.float32)
        print(f"{name}: reference compress+spmm(B=16) {dt:.1f}s")
    return out, ys


def main():
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small_cases())
    print("small.npz written")
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **cfg1_case())
    print("cfg1.npz written")
    large, ys = large_cases()
    with open(os.path.join(HERE, "large.json"), "w") as fh:
        json.dump(large, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "large_y.npz"), **ys)
    print("large.json written")


if __name__ == "__main__":
    main()
