"""Stream order under programmatic dependent launch: the compressor's chain (each kernel waits for
its predecessor) and the SpMM's early weight streams, back to back on one stream without host
synchronisation, reusing the cached per-stream workspace -- every result equal to the same call
made alone."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_20496_b200 as H  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _fields(p):
    """every array of the pack, the operand image up to its used length (capacities are padded)"""
    kp, eb = int(p.tile_kofs[-1]), int(p.tile_eofs[-1])
    return [p.tile_ptr, p.vec_idx, p.nm_pos, p.kept, p.tile_kofs, p.tile_eofs, p.gidx[:kp],
            p.a_vals[:kp * p.V // 2], p.a_meta[:eb * p.V * 4]]


def test_back_to_back_compress_and_spmm_match_isolated_calls():
    m, n, B = 1024, 2048, 512
    cfg = H.HiNMConfig(64, 2, 4, 0.5)
    gen = torch.Generator(device="cuda").manual_seed(5)
    Ws = [torch.randn(m, n, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3)]
    X = torch.randn(n, B, generator=gen, device="cuda").to(torch.bfloat16)
    sos = [np.random.default_rng(10 + i).permutation(m) for i in range(3)]
    # isolated: synchronise around every call
    ref_packs, ref_y = [], []
    for W, so in zip(Ws, sos):
        torch.cuda.synchronize()
        p = H.compress(W, cfg, so, groups=False)
        torch.cuda.synchronize()
        ref_packs.append(p)
        ref_y.append(H.spmm(p, X, order="original").clone())
        torch.cuda.synchronize()
    # back to back: compress, SpMM, compress, SpMM, ... with no host synchronisation
    packs, ys = [], []
    for W, so in zip(Ws, sos):
        p = H.compress(W, cfg, so, groups=False)
        packs.append(p)
        ys.append(H.spmm(p, X, order="original"))
    torch.cuda.synchronize()
    for i, (p, r) in enumerate(zip(packs, ref_packs)):
        for a, b in zip(_fields(p), _fields(r)):
            assert torch.equal(a, b), f"pack {i}"
        assert torch.equal(ys[i], ref_y[i]), f"spmm {i}"
