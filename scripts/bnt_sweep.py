"""Per-tile image: time at the library's token-unit choice under HINM_BN (128 | 256 | unset).

    HINM_BN=128 python scripts/bnt_sweep.py > a.jsonl     (one process per setting: knobs are read once)
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cfg_images import timed

dev = torch.device("cuda")
SHAPES = [(768, 768), (3072, 768), (768, 3072), (4096, 4096), (11008, 4096), (4096, 11008), (2048, 512), (512, 2048)]
TOKENS = [256, 512, 1024, 2048, 4096]
for i, (m, n) in enumerate(SHAPES):
    g = torch.Generator(device=dev).manual_seed(7 + i)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    for V, sv in ((64, 0.5), (128, 0.5), (64, 0.75)):
        pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), np.random.default_rng(i).permutation(m), groups=False)
        for B in TOKENS:
            X = torch.randn(n, B, generator=g, device=dev).to(torch.bfloat16)
            Y = torch.empty(m, B, dtype=torch.bfloat16, device=dev)
            us = timed(lambda: H.spmm(pack, X, out=Y, order="original", image="tiles"), True)
            print(json.dumps({"m": m, "n": n, "V": V, "sv": sv, "B": B, "T": pack.T, "k_t": pack.total_keep / pack.T,
                              "bn": os.environ.get("HINM_BN", "auto"), "us": round(us, 2)}), flush=True)
        del pack
