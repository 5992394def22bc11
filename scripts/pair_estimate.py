"""Experiment: what would a tile-pair operand image (two V=64 tiles on one M=128 instruction over
the union of their kept sets, DESIGN 4.1) run at on the LLaMA FFN shapes?  Emulated with the
existing M=128 path: V=128 at s_v=0 (every 128-row tile runs K = n positions, ~= the pair's
0.96 x 2 k_bar) and, with HINM_GATHER=dbg_pad_quarter, every 4th row left unfetched (the pair's
~22-25 % zero-filled padding).  Prints the V=64 kernel beside it.

    python scripts/pair_estimate.py                               # V=64 s_v=0.5 and V=128 s_v=0
    HINM_GATHER=dbg_pad_quarter python scripts/pair_estimate.py   # (timing only)
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

tok = 16384
dev = torch.device("cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
out = {"variant": os.environ.get("HINM_GATHER", "default")}
for name, m, n in (("up", 11008, 4096), ("down", 4096, 11008)):
    g = torch.Generator(device=dev).manual_seed(1)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    X = torch.randn(n, tok, generator=g, device=dev).to(torch.bfloat16)
    Y = torch.empty(m, tok, dtype=torch.bfloat16, device=dev)
    so = np.random.default_rng(2).permutation(m)
    for V, sv in ((64, 0.5), (128, 0.0)):
        if m % V:
            continue
        pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), so)
        out[f"{name}_V{V}_sv{sv}"] = round(t(lambda: H.spmm(pack, X, out=Y, order="original")), 4)
        del pack
print(json.dumps(out), flush=True)
