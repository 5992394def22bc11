"""Per-stage event trace of CTA pair 0 in the CTA-pair SpMM (experiments build with -DHINM_TRACE):
where the ~1 k cycles per 128-K stage go.  python scripts/pair_trace.py m n tokens"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import _lib

m, n, tokens = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
lib = _lib.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m), groups=True)
X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    H.spmm(pack, X, out=Y, image="groups")
torch.cuda.synchronize()
buf = np.zeros((11, 1024), np.uint64)
lib.hinm_exp_trace.argtypes = [ctypes.c_void_p]
assert lib.hinm_exp_trace(buf.ctypes.data) == 0
t = buf.astype(np.float64)
off = t[10][1] - t[10][0]
L0 = t[10][0]
Lfull, Lafull, Lpfull = t[0] - L0, t[1] - L0, t[2] - L0
Pfull, Pafull = t[3] - off - L0, t[4] - off - L0
Lgo, Pgo = t[5] - L0, t[6] - off - L0
LAgo, PAgo = t[7] - L0, t[8] - off - L0
S = int(np.count_nonzero(t[2]))
S = min(S, 1024) - 8
rng = slice(40, S)
md = lambda a: float(np.median(a[rng]))
print(f"stages traced {S}; peer clock offset {off:.0f}")
d = np.diff(Lpfull)[40:S]
print(f"issue interval (L_pfull[i+1]-L_pfull[i])        median {float(np.median(d)):8.0f} mean {float(d.mean()):8.0f} "
      f"p90 {float(np.percentile(d, 90)):8.0f} p99 {float(np.percentile(d, 99)):8.0f}")
big = np.nonzero(d > 1500)[0] + 40
print("stages after gaps > 1500 clk:", big[:40].tolist())
for i in big[:6]:
    print(f"  gap at {i}->{i+1}: {d[i-40]:.0f}; L_go {Lgo[i+1]-Lpfull[i]:.0f} L_full {Lfull[i+1]-Lpfull[i]:.0f} "
          f"L_afull {Lafull[i+1]-Lpfull[i]:.0f} P_full {Pfull[i+1]-Lpfull[i]:.0f} P_afull {Pafull[i+1]-Lpfull[i]:.0f} "
          f"LA_go {LAgo[i+1]-Lpfull[i]:.0f} PA_go {PAgo[i+1]-Lpfull[i]:.0f}")
print(f"leader fill latency  (L_full - L_go)             {md(Lfull - Lgo):8.0f}")
print(f"peer fill latency    (P_full - P_go)             {md(Pfull - Pgo):8.0f}")
print(f"leader: pfull after full                          {md(Lpfull - Lfull):8.0f}")
print(f"leader: afull after full                          {md(Lafull - Lfull):8.0f}")
print(f"peer full vs leader full (P_full - L_full)        {md(Pfull - Lfull):8.0f}")
print(f"relay: L_pfull - P_afull (relay + hop)            {md(Lpfull - Pafull):8.0f}")
print(f"peer afull after peer full                        {md(Pafull - Pfull):8.0f}")
print(f"gather restart after issue (L_go[i+4]-L_pfull[i]) {float(np.median((Lgo[4:] - Lpfull[:-4])[40:S])):8.0f}")
print(f"peer restart after issue (P_go[i+4]-L_pfull[i])   {float(np.median((Pgo[4:] - Lpfull[:-4])[40:S])):8.0f}")
print(f"A go lead over X go (L_go - LA_go)                {md(Lgo - LAgo):8.0f}")
print(f"fraction of stages where peer later than leader  {float(np.mean((Pafull > np.maximum(Lfull, Lafull))[rng])):8.2f}")
for i in range(60, 72):
    print(i, int(Lgo[i]), int(Lfull[i]), int(Lafull[i]), int(Lpfull[i]), "| peer", int(Pgo[i]), int(Pfull[i]), int(Pafull[i]))
