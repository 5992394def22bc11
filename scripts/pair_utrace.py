"""Per-CTA unit timeline of one SpMM launch (experiments build with -DHINM_TRACE): globaltimer at
kernel start and at every unit's accumulator commit (MMA warp) -> per-CTA span, unit durations,
tail.  python scripts/pair_utrace.py m n tokens image"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import _lib

m, n, tokens, image = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
lib = _lib.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.random.default_rng(2).permutation(m), groups=True)
X = torch.randn(n, tokens, generator=g, device=dev).to(torch.bfloat16)
Y = torch.empty(m, tokens, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    H.spmm(pack, X, out=Y, image=image)
torch.cuda.synchronize()
buf = np.zeros((160, 72), np.uint64)
lib.hinm_exp_utrace.argtypes = [ctypes.c_void_p]
lib.hinm_exp_utrace(buf.ctypes.data)
t = buf.astype(np.float64)
starts = t[:, 0]
valid = starts > 0
t0 = starts[valid].min()
rows = []
for c in range(160):
    if not valid[c]:
        continue
    u = t[c, 1:]
    u = u[u > 0]
    if len(u) == 0:
        continue
    rows.append((c, (starts[c] - t0) / 1e3, (u[-1] - t0) / 1e3, len(u), np.median(np.diff(u)) / 1e3 if len(u) > 2 else 0))
rows = np.array(rows)
print(f"{image}: CTAs with units {len(rows)}; start spread {rows[:,1].max():.2f} us; end min {rows[:,2].min():.2f} "
      f"median {np.median(rows[:,2]):.2f} max {rows[:,2].max():.2f} us; units/CTA {int(rows[:,3].min())}-{int(rows[:,3].max())}; "
      f"median unit {np.median(rows[:,4]):.2f} us (min {rows[:,4].min():.2f}, max {rows[:,4].max():.2f})")
first = (t[valid, 1] - t0) / 1e3
print(f"first unit done: median {np.median(first):.2f} us, max {first.max():.2f}")
# effective SM clock: clock64 at start (trace row 8) vs at the last unit commit (row 9, slot (units & 3))
tr = np.zeros((11, 1024), np.uint64)
lib.hinm_exp_trace.argtypes = [ctypes.c_void_p]
lib.hinm_exp_trace(tr.ctypes.data)
for c in (0, 2, 10, 40):
    u = t[c, 1:]
    nu = int(np.count_nonzero(u))
    if nu < 2:
        continue
    ck_end = float(tr[9][c * 4 + (nu & 3)])
    ck0 = float(tr[8][c])
    ns = float(u[nu - 1] - t[c, 0])
    print(f"CTA {c}: {nu} units, {ns/1e3:.1f} us, {ck_end - ck0:.0f} clocks -> {(ck_end - ck0) / ns:.3f} GHz")
