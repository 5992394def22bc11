"""A/B: compress_layers side-stream count (1 / 2 / 3) and staggering (on / off) for the LLaMA FFN's
three layers: GPU time of
the call captured in a CUDA graph, L2 flushed before each replay (median of 9).

Measured (scripts/r04_gpu5.sh, two passes): 1 stream 0.358 / 0.361 ms, 2 streams 0.301 / 0.301,
3 streams 0.243 / 0.248, staggered (layer i + 1 starting after layer i's score kernel, through a
hinm_compress_bf16_staged entry that recorded an event there) 2 streams 0.318 / 0.289, 3 streams
0.268 / 0.272: the chains in lockstep are fastest (three concurrent passes over W draw more HBM
bandwidth than one), so the staged entry and the `stagger` option were removed again.

    python scripts/layers_streams_ab.py
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2407_20496_b200 as H  # noqa: E402

dev = torch.device("cuda", 0)
cfg = H.HiNMConfig(64, 2, 4, 0.5)
Ws, sos = [], []
for i, (name, m, n) in enumerate(bench.layer_shapes()):
    g = torch.Generator(device=dev).manual_seed(1000 + i)
    Ws.append(torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16))
    sos.append(torch.randperm(m, generator=torch.Generator().manual_seed(2000 + i)).numpy())
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}
for rep in range(2):
    for ns, stg in ((1, False), (2, False), (3, False), (2, True), (3, True)):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            H.compress_layers(Ws, cfg, sos, groups=False, streams=ns, stagger=stg)
            with torch.cuda.graph(g, stream=s):
                H.compress_layers(Ws, cfg, sos, groups=False, streams=ns, stagger=stg)
        torch.cuda.current_stream().wait_stream(s)
        ts = []
        for _ in range(9):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out.setdefault(f"streams{ns}{'_stagger' if stg else ''}", []).append(round(statistics.median(ts), 4))
print(json.dumps(out))
