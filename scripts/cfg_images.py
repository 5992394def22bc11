"""Per-row time of both operand images (forced) vs the library's automatic pick, on a bench config.

    python scripts/cfg_images.py cfg4 [cfg4_875 cfg2 ...]
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2407_20496_b200 as H

dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timed(fn, graph, steps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            fn()
        torch.cuda.current_stream().wait_stream(st)
        with torch.cuda.graph(g):
            for _ in range(steps):
                fn()
        g.replay()
        run = g.replay
    else:
        def run():
            for _ in range(steps):
                fn()
    flush.fill_(1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3


for cfg in (sys.argv[1:] if __name__ == "__main__" else []):  # importable for timed()
    for i, (label, m, n, tokens, v, sv, count, graph) in enumerate(bench.cfg_cases(cfg)):
        g = torch.Generator(device=dev).manual_seed(31 + i)
        W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
        X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
        Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
        pack = H.compress(W, H.HiNMConfig(v, 2, 4, sv), np.random.default_rng(i).permutation(m))
        row = {"cfg": cfg, "gemm": label, "m": m, "n": n, "tokens": tokens, "V": v, "sv": float(sv),
               "T": pack.T, "k_t": pack.total_keep / pack.T}
        if pack.group is not None:
            row["gT"] = pack.group.T
            row["K_u"] = pack.group.total_keep / pack.group.T
        for img in ("auto", "tiles", "groups"):
            if img == "groups" and pack.group is None:
                continue
            row[img] = round(timed(lambda: H.spmm(pack, X, out=Y, order="original", image=img), graph), 1)
        row["cublas"] = round(timed(lambda: torch.matmul(W, X, out=Y), graph), 1)
        print(json.dumps(row), flush=True)
        del W, X, Y, pack
