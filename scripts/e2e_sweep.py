"""End-to-end (host buffers) sweep of the HostChain chunk size on the bench workload, plus raw
pinned H2D / D2H bandwidth (contiguous and the chain's 2-D strided pattern)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H

dev = torch.device("cuda")
tok = 16384
cfg = H.HiNMConfig(64, 2, 4, 0.5)
packs = {}
for i, (nm, m, n) in enumerate((("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008))):
    g = torch.Generator(device=dev).manual_seed(1000 + i)
    W = torch.randn(m, n, generator=g, device=dev).to(torch.bfloat16)
    packs[nm] = H.compress(W, cfg, np.random.default_rng(2000 + i).permutation(m))
xh = torch.randn(4096, tok).to(torch.bfloat16).pin_memory()
yh = torch.empty(4096, tok, dtype=torch.bfloat16).pin_memory()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, it=10):
    for _ in range(2): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
out = {}
xd = torch.empty(4096, tok, dtype=torch.bfloat16, device=dev)
out["h2d_contig_gbs"] = round(xh.numel() * 2 / t(lambda: xd.copy_(xh, non_blocking=True)) / 1e6, 1)
out["d2h_contig_gbs"] = round(xh.numel() * 2 / t(lambda: yh.copy_(xd, non_blocking=True)) / 1e6, 1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
xd2 = torch.empty_like(xd)
def duplex():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(xd2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
out["duplex_each_gbs"] = round(xh.numel() * 2 / t(duplex) / 1e6, 1)
for chunk in (1024, 2048, 4096):
    ch = H.HostChain([(packs["gate"], 0, 1, "original"), (packs["up"], 0, 2, "original"),
                      (packs["down"], 2, 3, "original")], out_buf=3, chunk=chunk, device=dev)
    out[f"e2e_ms_chunk{chunk}"] = round(t(lambda: ch.run(xh, yh)), 4)
print(json.dumps(out))
# diagnostics: the chain's compute alone (device buffers, 2048-token chunks) and the copy pipeline alone
if os.environ.get("E2E_DIAG"):
    xc = torch.empty(4096, 2048, dtype=torch.bfloat16, device=dev).normal_()
    def comp():
        for _ in range(tok // 2048):
            g = H.spmm(packs["gate"], xc, order="original")
            u = H.spmm(packs["up"], xc, order="original")
            H.spmm(packs["down"], u, order="original")
    out["compute_only_ms_chunk2048"] = round(t(comp), 4)
    print(json.dumps(out))
    # the duplex copies alone and with the chain's compute running concurrently on a third stream
    s3 = torch.cuda.Stream()
    def duplex_with_compute():
        with torch.cuda.stream(s3):
            comp()
        duplex()
        torch.cuda.current_stream().wait_stream(s3)
    out["duplex_plus_compute_ms"] = round(t(duplex_with_compute), 4)
    out["duplex_ms"] = round(t(duplex), 4)
    print(json.dumps(out))
