"""SpMM time over a sustained run with NVML clock / power samples (experiment)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, pynvml
import paper_2407_20496_b200 as H

dev = torch.device("cuda")
m, n, tok = 11008, 4096, 16384
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m))
X = torch.randn(n, tok, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, tok, dtype=torch.bfloat16, device=dev)
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()
def poll():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)
th = threading.Thread(target=poll, daemon=True); th.start()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
t0 = time.perf_counter()
for rep in range(40):
    s.record()
    for _ in range(10):
        H.spmm(pack, X, out=Y)
    e.record(); torch.cuda.synchronize()
    res.append((round(time.perf_counter() - t0, 3), round(s.elapsed_time(e) / 10, 4)))
stop.set(); th.join()
for tt, ms in res[::3]:
    near = [x for x in samples if abs(x[0] - t0 - tt) < 0.01]
    c = near[-1] if near else samples[-1]
    print(f"t={tt:6.3f}s  {ms:.4f} ms  sm={c[1]} MHz  power={c[2]:.0f} W  reasons=0x{c[3]:x}")
