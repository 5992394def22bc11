"""Small end-to-end run for compute-sanitizer (memcheck / synccheck / racecheck): compressor +
tcgen05 SpMM at V in {32, 64, 128}, both output orders, ragged tokens, an empty tile."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import synth

for V, m, n, B in ((64, 256, 512, 264), (32, 128, 256, 64), (128, 256, 384, 136)):
    W = torch.as_tensor(synth.randn_bf16((m, n), V)).to("cuda", torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), synth.random_sigma_o(m, V + 1))
    X = torch.as_tensor(synth.randn_bf16((n, B), V + 2)).to("cuda", torch.bfloat16)
    for order in ("sigma", "original"):
        Y = H.spmm(pack, X, order=order)
        R = H.spmm_simt(pack, X, order=order)
        torch.cuda.synchronize()
        err = (Y.float() - R).abs().max().item() / max(R.abs().max().item(), 1e-30)
        assert err < 1e-2, err
print("sanitize smoke ok")
