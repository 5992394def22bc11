"""Per-tile vs union-group image over token counts (calibration of the per-call choice in
hinm_spmm_bf16): python scripts/pair_sweep.py  -> one JSON line per (shape, tokens)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

dev = torch.device("cuda")
shapes = [("up", 11008, 4096, 64, 0.5), ("down", 4096, 11008, 64, 0.5), ("bert_ffn1", 3072, 768, 64, 0.5),
          ("bert_ffn2", 768, 3072, 64, 0.5), ("bert_qkvo", 768, 768, 64, 0.5), ("sq_v32", 4096, 4096, 32, 0.5),
          ("sq_v64_k25", 4096, 4096, 64, 0.75)]
toks = [256, 512, 1024, 2048, 4096, 8192, 16384]


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name, m, n, V, sv in shapes:
    gen = torch.Generator(device=dev).manual_seed(1)
    W = torch.randn(m, n, generator=gen, device=dev).to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), np.random.default_rng(2).permutation(m), groups=True)
    for B in toks:
        X = torch.randn(n, B, generator=gen, device=dev).to(torch.bfloat16)
        Y = torch.empty(m, B, dtype=torch.bfloat16, device=dev)
        r = {"shape": name, "m": m, "n": n, "V": V, "s_v": sv, "tokens": B}
        r["tiles_us"] = round(1e3 * timeit(lambda: H.spmm(pack, X, out=Y, image="tiles")), 2)
        r["groups_us"] = round(1e3 * timeit(lambda: H.spmm(pack, X, out=Y, image="groups")), 2)
        r["auto_us"] = round(1e3 * timeit(lambda: H.spmm(pack, X, out=Y)), 2)
        r["cublas_us"] = round(1e3 * timeit(lambda: torch.matmul(W, X)), 2)
        r["K_tile"] = pack.total_keep // pack.T
        r["K_union"] = pack.group.total_keep // pack.group.T
        print(json.dumps(r), flush=True)
