"""GPU: the end-to-end host-buffer chain (hinm_chain_run_host) against the device path.

Chunking the tokens does not change any token's accumulation order, so with the operand image
fixed (per-tile or union-group) the chain's output must be bit-identical to the device SpMMs on
the whole batch; the device path itself is checked against the oracle in test_gpu_parity.py and
test_gpu_group.py.  Covers ragged chunks, a two-layer chain with the
sigma_o restore fused, SIGMA order, and the argument checks.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _pack(m, n, seed, V=64):
    W = torch.as_tensor(synth.randn_bf16((m, n), seed)).to("cuda", torch.bfloat16)
    return H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), synth.random_sigma_o(m, seed + 1))


@pytest.mark.parametrize("B,chunk", [(512, 128), (1000, 256), (2048, 2048), (8, 64), (1536, 512)])
def test_chain_matches_device_path(B, chunk):
    up = _pack(512, 256, 10)
    gate = _pack(512, 256, 20)
    down = _pack(256, 512, 30)
    X = torch.as_tensor(synth.randn_bf16((256, B), 5)).to(torch.bfloat16)
    for image in ("tiles", "groups"):  # the image is fixed: per-call choices could differ per chunk
        chain = H.HostChain([(gate, 0, 1, "original"), (up, 0, 2, "original"),
                             (down, 2, 3, "original")], out_buf=3, chunk=chunk, image=image)
        Yh = chain.run(X.pin_memory())
        torch.cuda.synchronize()
        Xd = X.cuda()
        ref = H.spmm(down, H.spmm(up, Xd, order="original", image=image), order="original", image=image)
        assert torch.equal(Yh, ref.cpu()), image


def test_chain_sigma_order_and_unpinned_host():
    p = _pack(256, 512, 40, V=32)
    X = torch.as_tensor(synth.randn_bf16((512, 264), 6)).to(torch.bfloat16)
    chain = H.HostChain([(p, 0, 1, "sigma")], out_buf=1, chunk=64)
    Yh = chain.run(X)                   # pageable host memory still works (no overlap)
    torch.cuda.synchronize()
    assert torch.equal(Yh, H.spmm(p, X.cuda(), order="sigma").cpu())


def test_chain_errors():
    p = _pack(256, 512, 50)
    with pytest.raises(H.ShapeMismatch):
        H.HostChain([(p, 0, 1, "original"), (p, 0, 1, "original"), (p, 1, 2, "original")],
                    out_buf=2)
    chain = H.HostChain([(p, 0, 1, "original")], out_buf=1, chunk=64)
    with pytest.raises(H.ShapeMismatch):
        chain.run(torch.zeros(100, 64, dtype=torch.bfloat16))
    with pytest.raises(ValueError):
        chain.run(torch.zeros(512, 12, dtype=torch.bfloat16))   # B % 8 != 0
