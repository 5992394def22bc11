"""Reproduce bench.py's compressor timing on its exact inputs (seeds 1000+i, torch.randn on the
device, torch.randperm sigma_o) and time each call -- used to chase a slow down-projection call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_20496_b200 as H

dev = torch.device("cuda", 0)
shapes = [("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]
dense, sos = {}, {}
for i, (name, m, n) in enumerate(shapes):
    g = torch.Generator(device=dev).manual_seed(1000 + i)
    dense[name] = torch.randn(m, n, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    sos[name] = torch.randperm(m, generator=torch.Generator().manual_seed(2000 + i)).numpy()
cfg = H.HiNMConfig(64, 2, 4, 0.5)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for rep in range(reps):
    for name, _, _ in shapes:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        H.compress(dense[name], cfg, sos[name])
        torch.cuda.synchronize()
        print(f"rep {rep} {name}: {(time.perf_counter() - t0) * 1e3:.3f} ms", flush=True)
