"""One compression of a LLaMA FFN shape (for ncu): python scripts/compress_once.py [up|down]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

m, n = (11008, 4096) if (sys.argv[1:] or ["up"])[0] == "up" else (4096, 11008)
g = torch.Generator(device="cuda").manual_seed(1)
W = torch.randn(m, n, generator=g, device="cuda").to(torch.bfloat16)
so = np.random.default_rng(2).permutation(m)
H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), so, groups=False)
torch.cuda.synchronize()
