"""Experiment: how much of the small-shape (cfg1 / cfg2) times is host launch overhead?

Times the same SpMM and torch.matmul three ways: eager back-to-back calls, one CUDA graph
holding ITERS calls, and the host cost of one eager call with the GPU idle.

    python scripts/host_overhead.py
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2407_20496_b200 as H  # noqa: E402

DEV = torch.device("cuda")
ITERS = 50


def ev_time(fn, iters=ITERS):
    torch.cuda.synchronize()
    time.sleep(0.3)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def graph_time(fn, iters=ITERS):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    time.sleep(0.3)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def host_time(fn, iters=200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / iters * 1e6


def main():
    for m, n, tok in ((768, 768, 4096), (3072, 768, 4096), (768, 3072, 4096), (768, 3072, 512),
                      (3072, 768, 512), (256, 64, 802816), (11008, 4096, 2048)):
        g = torch.Generator(device=DEV).manual_seed(0)
        W = torch.randn(m, n, generator=g, device=DEV).to(torch.bfloat16)
        X = torch.randn(n, tok, generator=g, device=DEV).to(torch.bfloat16)
        Y = torch.empty(m, tok, dtype=torch.bfloat16, device=DEV)
        Yc = torch.empty(m, tok, dtype=torch.bfloat16, device=DEV)
        pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(0).permutation(m))
        sp = lambda: H.spmm(pack, X, out=Y, order="original")
        cb = lambda: torch.matmul(W, X, out=Yc)
        print(f"{m}x{n} @ {tok}: spmm eager {ev_time(sp):8.2f} us graph {graph_time(sp):8.2f} us "
              f"host {host_time(sp):6.2f} us | cublas eager {ev_time(cb):8.2f} us graph "
              f"{graph_time(cb):8.2f} us host {host_time(cb):6.2f} us", flush=True)


if __name__ == "__main__":
    main()
