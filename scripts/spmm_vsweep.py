"""HiNM SpMM vs cuBLAS on a 4096x4096 GEMM for V in {32, 64, 128} x vector-keep {50%, 25%}
(BASELINE.json configs[4] shape, single GPU; tokens as argv[1])."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = n = 4096
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
cb = t(lambda: torch.matmul(W, X))
rows = []
for V in (32, 64, 128):
    for sv in (0.5, 0.75):
        pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), np.random.default_rng(2).permutation(m))
        ms = t(lambda: H.spmm(pack, X, out=Y))
        rows.append({"V": V, "s_v": sv, "ms": round(ms, 4), "cublas_ms": round(cb, 4),
                     "speedup": round(cb / ms, 3), "eff_tflops": round(2 * m * n * tokens / ms / 1e9, 1)})
print(json.dumps({"tokens": tokens, "variant": os.environ.get("HINM_GATHER", "default"), "rows": rows}))
