"""Time the gyro-permutation search on cfg1 (768x3072 BERT-base FFN, V=64, 2:4, s_v=0.5) with the
reference's default budgets (OCP 20 iterations, ICP up to 50 per tile).  The reference needs
~422 s per ICP iteration of one tile -- tens of hours for this run."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import permutation as P, synth

m, n = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (768, 3072)
ocp = int(sys.argv[3]) if len(sys.argv) > 3 else 20
W = synth.randn_bf16((m, n), 0).astype(np.float64)
cfg = H.HiNMConfig(64, 2, 4, 0.5, ocp_max_iters=ocp, icp_max_iters=50, seed=0)
t_h = [0.0]
orig = P.hungarian
def timed_h(C):
    t0 = time.perf_counter(); a = orig(C); t_h[0] += time.perf_counter() - t0; return a
P.hungarian = timed_h
t0 = time.perf_counter()
sigma, masks, rep = P.gyro_permute(W, cfg)
dt = time.perf_counter() - t0
print(json.dumps({"shape": [m, n], "seconds": round(dt, 2), "hungarian_s": round(t_h[0], 2),
                  "ocp_iters": ocp, "icp_iters_per_tile": [len(l) - 1 for l in rep.icp_logs],
                  "retained": rep.retained_saliency, "no_perm_retained": rep.no_perm_retained,
                  "fallback": rep.fallback_used}))
