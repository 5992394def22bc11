"""SpMM time vs. the base-address alignment of X and Y (experiment): both carved out of one
pool at chosen offsets from a 32 MB-aligned base."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

dev = torch.device("cuda")
m, n, tok = 11008, 4096, 16384
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def t(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it

xb, yb = n * tok * 2, m * tok * 2
pool = torch.empty(xb + yb + (96 << 20), dtype=torch.uint8, device=dev)
base = (pool.data_ptr() + (32 << 20) - 1) // (32 << 20) * (32 << 20) - pool.data_ptr()
src = torch.randn(n, tok, generator=g, device=dev).to(torch.bfloat16)

def view(off, numel, rows, cols):
    return pool[base + off: base + off + numel * 2].view(torch.bfloat16).view(rows, cols)

cases = [(0, 0), (1 << 20, 0), (0, 1 << 20), (12345 * 512, 777 * 512), (512, 512)]
for xo, yo in cases + cases[::-1] + cases:
    X = view(xo, n * tok, n, tok)
    X.copy_(src)
    Y = view(xb + (8 << 20) + yo, m * tok, m, tok)
    print(f"X+{xo:>9} Y+{yo:>9}: {t(lambda: H.spmm(pack, X, out=Y)):.4f} ms", flush=True)
