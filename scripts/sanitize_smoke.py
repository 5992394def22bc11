"""Small end-to-end run for compute-sanitizer (memcheck / synccheck / racecheck): compressor (|W| and
external-saliency paths) + tcgen05 SpMM at V in {32, 64, 128}, both output orders, ragged tokens,
the operand-image decoder, the union-group image + CTA-pair SpMM, and the gyro search's GPU kernels
(OCP costs, k-means distances, ICP)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_20496_b200 as H
from paper_2407_20496_b200 import permutation as P, synth

for V, m, n, B in ((64, 256, 512, 264), (32, 128, 256, 64), (128, 256, 384, 136)):
    W = torch.as_tensor(synth.randn_bf16((m, n), V)).to("cuda", torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), synth.random_sigma_o(m, V + 1))
    X = torch.as_tensor(synth.randn_bf16((n, B), V + 2)).to("cuda", torch.bfloat16)
    for order in ("sigma", "original"):
        Y = H.spmm(pack, X, order=order)
        R = H.spmm_simt(pack, X, order=order)
        torch.cuda.synchronize()
        err = (Y.float() - R).abs().max().item() / max(R.abs().max().item(), 1e-30)
        assert err < 1e-2, err
    assert np.array_equal(pack.to_host_arrays("image")[2], pack.to_host_arrays("view")[2])
    S = np.random.default_rng(V).standard_normal((m, n))
    H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), synth.random_sigma_o(m, V + 1), saliency=S)
# the union-group image (plan + build kernels) and the CTA-pair SpMM (cluster of 2, remote barriers)
for V, m, n, B in ((64, 320, 512, 264), (32, 256, 384, 520)):
    W = torch.as_tensor(synth.randn_bf16((m, n), V + 5)).to("cuda", torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), synth.random_sigma_o(m, V + 6), groups=True)
    X = torch.as_tensor(synth.randn_bf16((n, B), V + 7)).to("cuda", torch.bfloat16)
    for order in ("sigma", "original"):
        Y = H.spmm(pack, X, order=order, image="groups")
        R = H.spmm_simt(pack, X, order=order)
        torch.cuda.synchronize()
        err = (Y.float() - R).abs().max().item() / max(R.abs().max().item(), 1e-30)
        assert err < 1e-2, err
    pack.group.to_host_arrays("image")
# the compressor's other tile-sort paths: n > 4096 (1024-thread CTAs, 8192 buckets) and tie-heavy
# scores (two magnitudes -> buckets beyond the limit -> bitonic network)
W = torch.as_tensor(synth.randn_bf16((64, 4608), 7)).to("cuda", torch.bfloat16)
H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), synth.random_sigma_o(64, 8))
Wt = torch.where(torch.rand(128, 1024, device="cuda") < 0.5, 1.0, 2.0).to(torch.bfloat16)
Wt[:, ::2] = 1.0
H.compress(Wt, H.HiNMConfig(64, 2, 4, 0.5), synth.random_sigma_o(128, 9))
# gyro search kernels on a small instance (OCP + k-means + ICP)
Wg = synth.randn_bf16((128, 64), 3).astype(np.float64)
P.gyro_permute(Wg, H.HiNMConfig(32, 2, 4, 0.5, ocp_max_iters=2, icp_max_iters=2, seed=1))
torch.cuda.synchronize()
print("sanitize smoke ok")
