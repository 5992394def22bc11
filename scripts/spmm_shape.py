"""Time one SpMM shape (experiments): python scripts/spmm_shape.py m n tokens [V] [s_v]."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

m, n, tok = (int(a) for a in sys.argv[1:4])
V = int(sys.argv[4]) if len(sys.argv) > 4 else 64
sv = float(sys.argv[5]) if len(sys.argv) > 5 else 0.5
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
X = torch.randn(n, tok, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, tok, dtype=torch.bfloat16, device=dev)
pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), np.random.default_rng(2).permutation(m))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
ms = t(lambda: H.spmm(pack, X, out=Y))
cb = t(lambda: torch.matmul(W, X))
print(json.dumps({"shape": [m, n, tok, V, sv], "variant": os.environ.get("HINM_GATHER", "default"),
                  "ms": round(ms, 4), "cublas_ms": round(cb, 4), "speedup": round(cb / ms, 3)}))
