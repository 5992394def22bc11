"""Experiment: where the host time of one device.compress call goes (LLaMA up projection).

    python scripts/compress_host_profile.py

Prints the per-call host wall (min of 50) and the top functions of a cProfile over 50 calls."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20496_b200 as H  # noqa: E402

m, n = 11008, 4096
W = torch.randn(m, n, device="cuda").to(torch.bfloat16)
so = np.random.default_rng(2).permutation(m)
cfg = H.HiNMConfig(64, 2, 4, 0.5)
keep = [H.compress(W, cfg, so, groups=False) for _ in range(3)]
torch.cuda.synchronize()
walls = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    keep.append(H.compress(W, cfg, so, groups=False))
    walls.append(time.perf_counter() - t0)
    keep.pop(0)
print(f"host wall per call: min {min(walls) * 1e6:.1f} us, median {sorted(walls)[25] * 1e6:.1f} us")
# the C call alone (hinm_compress_bf16: argument checks + the chain's launches)
from paper_2407_20496_b200 import _lib  # noqa: E402

lib = _lib.load()
raw = lib.hinm_compress_bf16
ctime = []


def timed_call(*a):
    t0 = time.perf_counter()
    r = raw(*a)
    ctime.append(time.perf_counter() - t0)
    return r


lib.hinm_compress_bf16 = timed_call
for _ in range(50):
    torch.cuda.synchronize()
    keep.append(H.compress(W, cfg, so, groups=False))
    keep.pop(0)
lib.hinm_compress_bf16 = raw
print(f"C call (hinm_compress_bf16) per call: min {min(ctime) * 1e6:.1f} us, median {sorted(ctime)[25] * 1e6:.1f} us")
# three layers through compress_layers, eager: host wall vs stream time (CUDA events)
Ws = [W, torch.randn(m, n, device="cuda").to(torch.bfloat16), torch.randn(n, m, device="cuda").to(torch.bfloat16)]
sos = [so, np.random.default_rng(3).permutation(m), np.random.default_rng(4).permutation(n)]
for _ in range(3):
    keep3 = H.compress_layers(Ws, cfg, sos, groups=False)
hw, sw = [], []
for _ in range(20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    keep3 = H.compress_layers(Ws, cfg, sos, groups=False)
    e1.record()
    hw.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    sw.append(e0.elapsed_time(e1))
print(f"compress_layers x3 eager: host {sorted(hw)[10] * 1e6:.1f} us, stream {sorted(sw)[10] * 1e3:.1f} us")
hw = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    keep3 = [H.compress(w, cfg, s_, groups=False) for w, s_ in zip(Ws, sos)]
    hw.append(time.perf_counter() - t0)
print(f"3 x compress eager, one stream: host {sorted(hw)[10] * 1e6:.1f} us")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    keep3 = H.compress_layers(Ws, cfg, sos, groups=False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    keep.append(H.compress(W, cfg, so, groups=False))
    keep.pop(0)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
