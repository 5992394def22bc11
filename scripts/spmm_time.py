"""Time the HiNM SpMM (one kernel) on LLaMA FFN shapes; prints one JSON line per shape.
Used for kernel-variant experiments (select with HINM_GATHER=cp4|cp8|tma2|tma4)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
iters = 20
dev = torch.device("cuda")
out = {"variant": os.environ.get("HINM_GATHER", "cp4"), "tokens": tokens}
for name, m, n in (("up", 11008, 4096), ("down", 4096, 11008)):
    g = torch.Generator(device=dev).manual_seed(1)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m))
    X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
    Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        H.spmm(pack, X, out=Y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        H.spmm(pack, X, out=Y)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    for _ in range(3):
        torch.matmul(W, X)
    s.record()
    for _ in range(iters):
        torch.matmul(W, X)
    e.record(); torch.cuda.synchronize()
    cb = s.elapsed_time(e) / iters
    out[name] = {"ms": round(ms, 4), "cublas_ms": round(cb, 4), "speedup": round(cb / ms, 3),
                 "eff_tflops": round(2 * m * n * tokens / ms / 1e9, 1)}
print(json.dumps(out), flush=True)
