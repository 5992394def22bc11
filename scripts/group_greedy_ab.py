"""Union-group build: time it and dump the group image (for the A / B of two first-fit kernels).

    python scripts/group_greedy_ab.py out.npz     # HINM_B200_LIB / HINM_GREEDY_SMEM select the kernel
    python scripts/group_greedy_ab.py --cmp a.npz b.npz
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    same = sorted(a.files) == sorted(b.files) and all(np.array_equal(a[k], b[k]) for k in a.files)
    print("identical group images:", same, {k: a[k].shape for k in a.files if k.endswith("tile_ptr")})
    sys.exit(0 if same else 1)
import torch
import paper_2407_20496_b200 as H
dev = torch.device("cuda")
out = {}
for nm, V, m, n in (("up", 64, 11008, 4096), ("down", 64, 4096, 11008), ("v32", 32, 4096, 4096)):
    g = torch.Generator(device=dev).manual_seed(1)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), np.random.default_rng(2).permutation(m), groups=False)
    H.build_group_image(pack)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        H.build_group_image(pack)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    gp = pack.group
    print(f"{nm}: group build {min(ts) * 1e3:.2f} ms, K_union per group {int(gp.tile_ptr[-1]) / gp.T:.0f}")
    for f in ("tile_ptr", "vec_idx", "nm_pos", "kept", "gidx", "a_vals", "a_meta", "tile_kofs"):
        out[f"{nm}_{f}"] = getattr(gp, f).cpu().view(torch.int16 if getattr(gp, f).dtype == torch.bfloat16 else getattr(gp, f).dtype).numpy()
np.savez(sys.argv[1], **out)
