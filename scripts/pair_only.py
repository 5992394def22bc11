"""Only the union-group (CTA-pair) SpMM on one shape, for ncu captures: python scripts/pair_only.py m n V sv tokens reps"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

m, n, V = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
sv, tokens, reps = float(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), np.random.default_rng(2).permutation(m), groups=True)
X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
for _ in range(reps):
    H.spmm(pack, X, out=Y, image="groups")
torch.cuda.synchronize()
