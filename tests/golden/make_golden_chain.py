"""Golden for the reference's own build_layer_chain (spmm.py:206-234) with its default search,
gyro_permute, on two small layers (reduced OCP / ICP budgets so the reference finishes in seconds).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_chain.py

Writes tests/golden/chain_gyro.npz: per layer sigma_o, vector_index / nm_index / kept_values, and the
chain output compose_layers(chain, X) (spmm.py:237-244).  Inputs come from
paper_2407_20496_b200.synth (seeds below).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import hinm  # noqa: E402  (the reference)
from hinm.spmm import build_layer_chain, compose_layers  # noqa: E402

from paper_2407_20496_b200 import synth  # noqa: E402


def main():
    cfg = hinm.HiNMConfig(vector_size=32, nm_keep=2, nm_group=4, vector_sparsity=0.5, ocp_max_iters=3,
                          icp_max_iters=3, seed=5)
    W1 = synth.randn_bf16((128, 96), 51).astype(np.float64)
    W2 = synth.randn_bf16((64, 128), 52).astype(np.float64)
    X = synth.randn_bf16((96, 16), 53).astype(np.float64)
    chain = build_layer_chain([W1, W2], cfg)
    out = {"Y": compose_layers(chain, X), "final_sigma_o": np.asarray(chain.final_sigma_o, np.int64)}
    for l, e in enumerate(chain.layers):
        out[f"l{l}_sigma_o"] = np.asarray(e.sigma_o, np.int64)
        out[f"l{l}_vi"] = np.concatenate([t.vector_index for t in e.tiles])
        out[f"l{l}_nm"] = np.concatenate([t.nm_index.ravel() for t in e.tiles])
        out[f"l{l}_kv"] = np.concatenate([t.kept_values.ravel() for t in e.tiles])
    np.savez_compressed(os.path.join(HERE, "chain_gyro.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
