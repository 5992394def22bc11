"""Experiment: GPU-side time of the SpMM on the latency / epilogue-bound shapes (cfg1, cfg2, the
small-K cfg4 layers), CUDA-graph replays of ITERS calls so host launch overhead is excluded.
Kernel variants are selected with the HINM_* environment switches of hinm_spmm_bf16.

    python scripts/small_shapes.py [--cublas] [--sigma]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2407_20496_b200 as H  # noqa: E402

DEV = torch.device("cuda")
ITERS = 40
SHAPES = [(768, 3072, 512), (3072, 768, 512), (768, 768, 4096), (3072, 768, 4096),
          (768, 3072, 4096), (256, 64, 802816), (512, 128, 200704), (512, 256, 200704),
          (1024, 256, 50176), (2048, 512, 12544), (64, 576, 802816), (4096, 11008, 2048)]


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
    time.sleep(0.2)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    cublas = "--cublas" in sys.argv
    order = "sigma" if "--sigma" in sys.argv else "original"
    tag = {k: v for k, v in os.environ.items() if k.startswith("HINM_")}
    for m, n, tok in SHAPES:
        g = torch.Generator(device=DEV).manual_seed(0)
        W = torch.randn(m, n, generator=g, device=DEV).to(torch.bfloat16)
        X = torch.randn(n, tok, generator=g, device=DEV).to(torch.bfloat16)
        Y = torch.empty(m, tok, dtype=torch.bfloat16, device=DEV)
        pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(0).permutation(m))
        row = {"shape": f"{m}x{n}@{tok}", "spmm_us": round(graph_time(lambda: H.spmm(pack, X, out=Y, order=order)), 2)}
        if cublas:
            Yc = torch.empty(m, tok, dtype=torch.bfloat16, device=DEV)
            row["cublas_us"] = round(graph_time(lambda: torch.matmul(W, X, out=Yc)), 2)
        row.update(tag)
        row["order"] = order
        print(json.dumps(row), flush=True)
        del W, X, Y, pack
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
