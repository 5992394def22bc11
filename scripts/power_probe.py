"""Sustained power / SM clock of one kernel looped for ~2 s (NVML, 20 ms samples): union-group SpMM,
per-tile SpMM, cuBLAS dense, on the LLaMA up projection at 16384 tokens."""
import os, sys, threading, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, pynvml
import paper_2407_20496_b200 as H

pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
m, n, B = 11008, 4096, 16384
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m), groups=True)
X = torch.randn(n, B, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, B, dtype=torch.bfloat16, device=dev)


def run(name, fn, secs=2.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    samples, stop = [], [False]

    def sampler():
        while not stop[0]:
            samples.append((pynvml.nvmlDeviceGetPowerUsage(hd) / 1e3,
                            pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.02)

    th = threading.Thread(target=sampler)
    th.start()
    t0 = time.time()
    k = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < secs:
        for _ in range(20):
            fn()
        k += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    sm = samples[len(samples) // 4:]
    p = np.array([x[0] for x in sm]); c = np.array([x[1] for x in sm])
    print(json.dumps({"kernel": name, "ms": round(s.elapsed_time(e) / k, 4), "power_w_median": round(float(np.median(p)), 1),
                      "power_w_max": round(float(p.max()), 1), "sm_mhz_median": float(np.median(c)), "sm_mhz_min": float(c.min())}), flush=True)


run("groups", lambda: H.spmm(pack, X, out=Y, image="groups"))
run("tiles", lambda: H.spmm(pack, X, out=Y, image="tiles"))
run("cublas", lambda: torch.matmul(W, X, out=Y))
print(json.dumps({"power_limit_w": pynvml.nvmlDeviceGetEnforcedPowerLimit(hd) / 1e3}))
