"""Experiment: host-side cost of H.compress (LLaMA up 11008x4096) -- wall vs GPU stream time, and
the Python-side pieces before the C call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import device as D, model as Mo

dev = torch.device("cuda")
m, n = 11008, 4096
W = torch.randn(m, n, device=dev).to(torch.bfloat16)
so = np.random.default_rng(0).permutation(m)
cfg = H.HiNMConfig(64, 2, 4, 0.5)
for _ in range(3):
    H.compress(W, cfg, so)
torch.cuda.synchronize()

def t(name, fn, it=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:28s} host {(t1 - t0) / it * 1e6:8.1f} us   wall {(t2 - t0) / it * 1e6:8.1f} us", flush=True)

t("compress", lambda: H.compress(W, cfg, so))
so_t = torch.as_tensor(so, dtype=torch.int32, device=dev)
t("compress (sigma_o on device)", lambda: H.compress(W, cfg, so_t))
t("ensure_validated", lambda: Mo.ensure_validated(cfg, (m, n)))
t("sigma_o H2D", lambda: torch.as_tensor(np.asarray(so), dtype=torch.int32).to(dev))
vc = Mo.ensure_validated(cfg, (m, n))
t("_empty_pack", lambda: D._empty_pack(vc, dev))
p = D._empty_pack(vc, dev)
t("_alloc_operand_image", lambda: D._alloc_operand_image(p))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, arg in (("sigma host", so), ("sigma device", so_t)):
    torch.cuda.synchronize()
    s.record(); H.compress(W, cfg, arg); e.record(); torch.cuda.synchronize()
    print(f"stream time ({name}) {s.elapsed_time(e) * 1e3:8.1f} us")
