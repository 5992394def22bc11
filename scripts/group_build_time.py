"""Time the union-group image build per kernel (run under ncu --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
dev = torch.device("cuda")
for m, n in ((11008, 4096), (4096, 11008)):
    g = torch.Generator(device=dev).manual_seed(1)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m), groups=False)
    for _ in range(2):
        H.build_group_image(pack)
    torch.cuda.synchronize()
