"""Time the fused GPU compressor (hinm_compress_bf16) on the LLaMA FFN shapes."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = {}
for name, m, n in (("up", 11008, 4096), ("down", 4096, 11008)):
    g = torch.Generator(device="cuda").manual_seed(1)
    W = torch.randn(m, n, generator=g, device="cuda").to(torch.bfloat16)
    so = np.random.default_rng(2).permutation(m)
    cfg = H.HiNMConfig(64, 2, 4, 0.5)
    H.compress(W, cfg, so)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        H.compress(W, cfg, so)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    kbar = n // 2
    alg = 2 * m * n + m * kbar + m * kbar // 8 + 4 * (m // 64) * kbar + 4 * m
    best = min(ts)
    out[name] = {"ms": round(best * 1e3, 3), "algorithmic_bytes": alg, "gbs": round(alg / best / 1e9, 1)}
print(json.dumps(out))
