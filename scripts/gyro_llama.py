"""Gyro-permutation search at LLaMA-7B FFN scale with the reference's default budgets (SURVEY §8(f)
row 1): W = the up projection 11008 x 4096 (N(0,1) bf16-valued, seed 0), V = 64, 2:4, s_v = 0.5,
OCP 20 iterations (samples V/2 decaying 0.8x), ICP up to 50 iterations per tile, seed 0.

    python scripts/gyro_llama.py [m n ocp_iters] > gpurun_out/gyro_llama.json

Phase times come from wrapping the search's own entry points (ocp_iterate, icp_tile); the
reference needs ~422 s per ICP iteration of one cfg1 tile and materialises a 31 GB
k-means distance tensor per OCP round at this shape, i.e. it does not finish."""
import json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import permutation as P, synth

m, n = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (11008, 4096)
ocp = int(sys.argv[3]) if len(sys.argv) > 3 else 20
W = synth.randn_bf16((m, n), 0).astype(np.float64)
cfg = H.HiNMConfig(64, 2, 4, 0.5, ocp_max_iters=ocp, icp_max_iters=50, seed=0)
acc = {"ocp_s": 0.0, "icp_tile_s": 0.0, "ocp_costs_s": 0.0, "kmeans_s": 0.0, "hungarian_s": 0.0}
lock = threading.Lock()


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            with lock:
                acc[name] += time.perf_counter() - t0
    return w


P.ocp_iterate = timed("ocp_s", P.ocp_iterate)
P.icp_tile = timed("icp_tile_s", P.icp_tile)
P._ocp_costs = timed("ocp_costs_s", P._ocp_costs)
P.balanced_kmeans = timed("kmeans_s", P.balanced_kmeans)
P.hungarian = timed("hungarian_s", P.hungarian)
t0 = time.perf_counter()
sigma, masks, rep = P.gyro_permute(W, cfg)
dt = time.perf_counter() - t0
print(json.dumps({"shape": [m, n], "V": 64, "nm": "2:4", "s_v": 0.5, "ocp_iters": ocp, "icp_max_iters": 50,
                  "seconds": round(dt, 1), **{k: round(v, 1) for k, v in acc.items()},
                  "note": "icp_tile_s / hungarian_s are summed over 16 concurrent tile threads",
                  "icp_iters_per_tile_mean": round(float(np.mean([len(l) - 1 for l in rep.icp_logs])), 1),
                  "ocp_log_first_last": [rep.ocp_log[0], rep.ocp_log[-1]],
                  "retained": rep.retained_saliency, "no_perm_retained": rep.no_perm_retained,
                  "gain_vs_no_perm": rep.retained_saliency / rep.no_perm_retained - 1.0,
                  "fallback": rep.fallback_used}))
