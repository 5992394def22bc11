"""Energy split of the union-group SpMM (experiments build): sustained power x time of the full kernel
and of its timing-only variants (HINM_PAIR_DBG: 1 = no MMAs, 2 = no gather, 3 = no epilogue), LLaMA up
projection, 16384 tokens.  Each variant runs in a fresh process (the variant is read once)."""
import os, sys, subprocess, json
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, threading, time, json
sys.path.insert(0, "%s")
import numpy as np, torch, pynvml
import paper_2407_20496_b200 as H
pynvml.nvmlInit(); hd = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda"); g = torch.Generator(device=dev).manual_seed(1)
m, n, B = 11008, 4096, 16384
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m), groups=True)
X = torch.randn(n, B, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, B, dtype=torch.bfloat16, device=dev)
fn = lambda: H.spmm(pack, X, out=Y, image="groups")
for _ in range(3): fn()
torch.cuda.synchronize()
samples, stop = [], [False]
def sampler():
    while not stop[0]:
        samples.append((pynvml.nvmlDeviceGetPowerUsage(hd) / 1e3, pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.02)
th = threading.Thread(target=sampler); th.start()
t0 = time.time(); k = 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 2.0:
    for _ in range(20): fn()
    k += 20
    torch.cuda.synchronize()
e.record(); torch.cuda.synchronize(); stop[0] = True; th.join()
sm = samples[len(samples) // 4:]
p = float(np.median([x[0] for x in sm])); c = float(np.median([x[1] for x in sm]))
ms = s.elapsed_time(e) / k
print(json.dumps({"variant": os.environ.get("HINM_PAIR_DBG", "0"), "ms": round(ms, 4), "power_w": round(p, 1), "sm_mhz": c, "energy_mj": round(p * ms, 1)}))
''' % root
for v in ("0", "1", "2", "3"):
    env = dict(os.environ, HINM_PAIR_DBG=v, HINM_B200_LIB=os.path.join(root, "scripts", "libhinm_b200_exp.so"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:], flush=True)
