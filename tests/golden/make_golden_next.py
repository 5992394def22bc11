"""Golden vectors for the §8(f) rows, produced by the REAL reference package (build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_next.py

Writes (committed, small):
  tests/golden/io/config.json, encoding.json, permutation.json, report.json, chain.json
      files written by the reference's io.py writers (byte-compatibility of ours)
  tests/golden/next.npz
      shuffle_encoding(enc, default_rng(7)) outputs for a 2:4 and a 1:4 encoding,
      kept_triples counts, and a 2-layer build_layer_chain(no_perm_prune) / compose_layers run
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
from hinm import io as rio  # noqa: E402
from hinm.spmm import kept_triples, shuffle_encoding  # noqa: E402

from paper_2407_20496_b200 import synth  # noqa: E402


def encoding_for(m, n, cfg, seed):
    W = synth.randn_bf16((m, n), seed).astype(np.float64)
    sigma, masks, _ = hinm.no_perm_prune(W, cfg)
    return W, hinm.encode(W, masks, sigma, cfg)


def flat_tiles(prefix, enc, out):
    for t, tile in enumerate(enc.tiles):
        out[f"{prefix}t{t}_vi"] = np.asarray(tile.vector_index, dtype=np.int64)
        out[f"{prefix}t{t}_nm"] = np.asarray(tile.nm_index, dtype=np.int64)
        out[f"{prefix}t{t}_kv"] = np.asarray(tile.kept_values, dtype=np.float64)


def main():
    iod = os.path.join(HERE, "io")
    os.makedirs(iod, exist_ok=True)
    out = {}
    # --- io: files written by the reference
    cfg = hinm.HiNMConfig(vector_size=4, nm_keep=2, nm_group=4, vector_sparsity=0.5,
                          ocp_sample_schedule=(2, 1), seed=3)
    W, enc = encoding_for(16, 32, cfg, 11)
    with open(os.path.join(iod, "config.json"), "w", encoding="utf-8") as fh:
        json.dump(rio.config_to_dict(cfg), fh, indent=2, sort_keys=True)
        fh.write("\n")
    rio.save_encoding(enc, os.path.join(iod, "encoding.json"))
    sigma = hinm.GyroPermutation(sigma_o=np.asarray(enc.sigma_o),
                                 sigma_i=tuple(t.vector_index for t in enc.tiles))
    with open(os.path.join(iod, "permutation.json"), "w", encoding="utf-8") as fh:
        json.dump(rio.permutation_to_dict(sigma), fh, indent=2, sort_keys=True)
        fh.write("\n")
    rio.dump_json({"b": 1.0 / 3.0, "a": [np.float64(2.0) / 7.0, np.int64(5)], "c": {"z": 1e-12}},
                  os.path.join(iod, "report.json"))
    with open(os.path.join(iod, "chain.json"), "w", encoding="utf-8") as fh:
        json.dump({"layers": ["encoding.json", "encoding.json"]}, fh)
    # --- group-order freedom: the reference's shuffle with a fixed generator
    for tag, (m, n, N, M) in {"s24": (8, 32, 2, 4), "s14": (8, 32, 1, 4)}.items():
        c = hinm.HiNMConfig(vector_size=4, nm_keep=N, nm_group=M, vector_sparsity=0.5)
        Wt, e = encoding_for(m, n, c, 21)
        out[f"{tag}_W"] = Wt
        out[f"{tag}_meta"] = np.array([m, n, 4, N, M], dtype=np.int64)
        out[f"{tag}_sigma_o"] = np.asarray(e.sigma_o, dtype=np.int64)
        flat_tiles(f"{tag}_enc_", e, out)
        sh = shuffle_encoding(e, np.random.default_rng(7))
        flat_tiles(f"{tag}_sh_", sh, out)
        out[f"{tag}_ntriples"] = np.array(len(kept_triples(e)), dtype=np.int64)
    # --- chain: two layers, identity pipeline, run end to end by the reference
    c = hinm.HiNMConfig(vector_size=64, nm_keep=2, nm_group=4, vector_sparsity=0.5)
    W1 = synth.randn_bf16((256, 128), 31).astype(np.float64)
    W2 = synth.randn_bf16((128, 256), 32).astype(np.float64)
    X = synth.randn_bf16((128, 24), 33).astype(np.float64)
    # build_layer_chain (spmm.py:206-234) with the identity search: its loop, no_perm_prune
    from hinm.spmm import compose_layers
    from hinm.permutation import no_perm_prune

    layers, prev = [], None
    for Wl in (W1, W2):
        Wv = Wl if prev is None else Wl[:, prev]
        sig, masks, _ = no_perm_prune(Wv, c)
        layers.append(hinm.encode(Wv, masks, sig, c))
        prev = sig.sigma_o
    chain = hinm.LayerChain(layers=tuple(layers))
    out["chain_W1"], out["chain_W2"], out["chain_X"] = W1, W2, X
    out["chain_Y"] = compose_layers(chain, X)
    for l, e in enumerate(layers):
        out[f"chain_l{l}_sigma_o"] = np.asarray(e.sigma_o, dtype=np.int64)
        flat_tiles(f"chain_l{l}_", e, out)
    np.savez_compressed(os.path.join(HERE, "next.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
