"""Time the fused GPU compressor (hinm_compress_bf16 through device.compress) on the LLaMA FFN shapes.

    python scripts/compress_time.py [reps]

Per shape: host wall of one API call (min), stream time of one call (CUDA events around it, median),
the per-call stream time of `reps` back-to-back calls, and the GPU time of one compression with the
host out of the loop (the call captured once in a CUDA graph, replayed `reps` times between events;
L2 flushed before each replay) -- with the achieved fraction of HBM bandwidth for the algorithmic
bytes (2mn + m k + m k / 8 + 4 T k + 4m).
"""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pk = os.path.join(root, "MEASURED_PEAKS.json")
peak = json.load(open(pk))["hbm_gbs"] if os.path.exists(pk) else 6543.4
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for name, m, n in (("up", 11008, 4096), ("down", 4096, 11008)):
    g = torch.Generator(device="cuda").manual_seed(1)
    W = torch.randn(m, n, generator=g, device="cuda").to(torch.bfloat16)
    so = np.random.default_rng(2).permutation(m)
    cfg = H.HiNMConfig(64, 2, 4, 0.5)
    for _ in range(3):
        H.compress(W, cfg, so, groups=False)
    torch.cuda.synchronize()
    wall, stream = [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        H.compress(W, cfg, so, groups=False)
        e1.record()
        torch.cuda.synchronize()
        wall.append(time.perf_counter() - t0)
        stream.append(e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        H.compress(W, cfg, so, groups=False)
    e1.record()
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / reps
    # GPU time: the whole compression captured in one CUDA graph (host launch path removed)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        H.compress(W, cfg, so, groups=False)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="relaxed"):
        pack_g = H.compress(W, cfg, so, groups=False)
    graph.replay()
    torch.cuda.synchronize()
    gt = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        gt.append(e0.elapsed_time(e1))
    ref = H.compress(W, cfg, so, groups=False)
    same = all(torch.equal(getattr(ref, f), getattr(pack_g, f)) for f in ("tile_ptr", "vec_idx", "kept", "nm_pos",
                                                                            "tile_kofs", "tile_eofs"))
    kp = int(ref.tile_kofs[-1])
    same = same and torch.equal(ref.gidx[:kp], pack_g.gidx[:kp]) and torch.equal(ref.a_vals[:kp * 32], pack_g.a_vals[:kp * 32])
    kbar = n // 2
    alg = 2 * m * n + m * kbar + m * kbar // 8 + 4 * (m // 64) * kbar + 4 * m
    st = statistics.median(stream)
    gpu = statistics.median(gt)
    out[name] = {"wall_ms": round(min(wall) * 1e3, 3), "stream_ms": round(st, 3), "b2b_ms": round(b2b, 3),
                 "gpu_ms": round(gpu, 4), "graph_matches_eager": same,
                 "algorithmic_bytes": alg, "gbs_stream": round(alg / st / 1e6, 1),
                 "hbm_frac_stream": round(alg / st / 1e6 / peak, 4),
                 "hbm_frac_b2b": round(alg / b2b / 1e6 / peak, 4),
                 "hbm_frac_gpu": round(alg / gpu / 1e6 / peak, 4)}
    del graph
print(json.dumps(out))
