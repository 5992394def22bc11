"""Per-tile image vs union-group image (CTA-pair kernel) on the LLaMA FFN shapes and the cfg5 V sweep;
one JSON line per shape: ms of each image (CUDA events, 20 back-to-back launches), cuBLAS, group
build time, union K vs per-tile K."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
iters = 20
dev = torch.device("cuda")
shapes = [("up", 11008, 4096, 64, 0.5), ("down", 4096, 11008, 64, 0.5), ("sq_v64", 4096, 4096, 64, 0.5),
          ("sq_v32", 4096, 4096, 32, 0.5), ("sq_v64_k25", 4096, 4096, 64, 0.75), ("sq_v32_k25", 4096, 4096, 32, 0.75)]
if len(sys.argv) > 2:
    shapes = [s for s in shapes if s[0] in sys.argv[2].split(",")]


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name, m, n, V, sv in shapes:
    g = torch.Generator(device=dev).manual_seed(1)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, sv), np.random.default_rng(2).permutation(m), groups=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H.build_group_image(pack)
    torch.cuda.synchronize()
    tb = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    H.build_group_image(pack)
    torch.cuda.synchronize()
    tb2 = (time.perf_counter() - t0) * 1e3
    X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
    Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
    mt = timeit(lambda: H.spmm(pack, X, out=Y, image="tiles"))
    mg = timeit(lambda: H.spmm(pack, X, out=Y, image="groups"))
    ma = timeit(lambda: H.spmm(pack, X, out=Y))
    cb = timeit(lambda: torch.matmul(W, X))
    kt = pack.total_keep
    kg = pack.group.total_keep // 2
    print(json.dumps({"shape": name, "m": m, "n": n, "V": V, "s_v": sv, "tokens": tokens,
                      "tiles_ms": round(mt, 4), "groups_ms": round(mg, 4), "auto_ms": round(ma, 4),
                      "cublas_ms": round(cb, 4), "speedup_groups": round(cb / mg, 3),
                      "speedup_tiles": round(cb / mt, 3),
                      "eff_tflops_groups": round(2 * m * n * tokens / mg / 1e9, 1),
                      "group_build_ms": [round(tb, 2), round(tb2, 2)],
                      "K_tiles_per_256_rows": kt * 256 // m, "K_union_per_group": kg * 256 // max(1, pack.group.rows) if False else kg // max(1, pack.group.T // 2)}),
          flush=True)
