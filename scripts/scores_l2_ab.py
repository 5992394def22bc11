"""A/B: the score kernel's W loads evict_normal (product) vs evict_first (HINM_SCORES_STREAM=1 in the
experiments library).  GPU time of one compression per LLaMA FFN layer and of the three layers
through compress_layers (CUDA graphs, L2 flushed before each replay; bench.compress_gpu_ms).

    HINM_B200_LIB=scripts/libhinm_b200_exp.so [HINM_SCORES_STREAM=1] python scripts/scores_l2_ab.py

Measured in round 2 (scripts/r04_gpu3.sh, and r04_gpu6.sh for the HINM_SCORES_PIPE / _NT64 variants):
no difference; the knobs and the variants
were removed from compress.cu afterwards.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2407_20496_b200 as H  # noqa: E402

dev = torch.device("cuda", 0)
cfg = H.HiNMConfig(64, 2, 4, 0.5)
dense, sos = {}, {}
for i, (name, m, n) in enumerate(bench.layer_shapes()):
    g = torch.Generator(device=dev).manual_seed(1000 + i)
    dense[name] = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    sos[name] = torch.randperm(m, generator=torch.Generator().manual_seed(2000 + i)).numpy()
ref = {k: H.compress(dense[k], cfg, sos[k], groups=False) for k in dense}
out = bench.compress_gpu_ms(H, torch, dense, cfg, sos, reps=9)
again = {k: H.compress(dense[k], cfg, sos[k], groups=False) for k in dense}
same = all(torch.equal(ref[k].kept, again[k].kept) and torch.equal(ref[k].vec_idx, again[k].vec_idx) for k in ref)
import hashlib  # noqa: E402

digest = hashlib.sha256()
for k in sorted(ref):
    for f in ("tile_ptr", "vec_idx", "nm_pos", "kept", "a_vals"):
        digest.update(getattr(ref[k], f).view(torch.uint8).cpu().numpy().tobytes())
knobs = {k: v for k, v in os.environ.items() if k.startswith("HINM_SCORES")}
print(json.dumps({"knobs": knobs, "same_packs": same, "digest": digest.hexdigest()[:16],
                  **{k: round(v, 4) for k, v in out.items()}}))
