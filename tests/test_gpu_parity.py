"""GPU parity: the CUDA library (through the C ABI) against the pinned oracle / reference goldens.

Bit-exact: vector masks, survivors, vector_index, nm_index, kept values, element masks.
SpMM: rtol 1e-2 / atol 1e-3 against the reference's float64 result (bf16 in, fp32 accumulate,
bf16 out -- BASELINE.json north_star tolerance); the CUDA-core cross-check kernel (fp32 out)
must agree to 1e-5 relative.
"""

import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hinm_oracle as O  # noqa: E402
from conftest import GOLDEN, case, load_small  # noqa: E402

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import device as D  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402

Z, NAMES = load_small()
RTOL, ATOL = 1e-2, 1e-3


def _cfg(d):
    num, den = d["s_v"]
    from fractions import Fraction

    return H.HiNMConfig(d["V"], d["N"], d["M"], Fraction(num, den))


def _bf16_exact(W):
    return np.array_equal(synth.bf16_round(W.astype(np.float32)).astype(np.float64), W)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("key", NAMES)
def test_dropin_pruning_matches_reference(key):
    d = case(Z, key)
    cfg = _cfg(d)
    S = H.magnitude_saliency(d["W"])
    vm = H.vector_prune(S, cfg, d["sigma_o"])
    assert np.array_equal(vm, d["vector_mask"]), "vector mask"
    sigma = H.GyroPermutation(d["sigma_o"], tuple(d["sigma_i"]))
    em = H.nm_prune(S, vm, cfg, sigma)
    assert np.array_equal(em, d["element_mask"]), "element mask"
    enc = H.encode(d["W"], H.MaskPair(vm, em), sigma, cfg)
    vidx = np.concatenate([t.vector_index for t in enc.tiles])
    nmi = np.concatenate([t.nm_index.ravel() for t in enc.tiles])
    kv = np.concatenate([t.kept_values.ravel() for t in enc.tiles])
    assert np.array_equal(vidx, d["vector_index"])
    assert np.array_equal(nmi, d["nm_index"].astype(np.int64))
    assert np.array_equal(kv, d["kept_values"])
    assert np.array_equal(H.decode(enc, (d["m"], d["n"])), d["decode"])


@pytest.mark.parametrize("key", [k for k in NAMES if k.startswith(("rand", "kat_"))])
def test_fused_compressor_matches_reference(key):
    d = case(Z, key)
    if not _bf16_exact(d["W"]):
        pytest.skip("weights not bf16-representable")
    W = torch.as_tensor(d["W"].astype(np.float32)).cuda().to(torch.bfloat16)
    pack = H.compress(W, _cfg(d), d["sigma_o"], sigma_i=d["sigma_i"])
    tiles = pack.to_host_tiles()
    assert np.array_equal(np.concatenate([t[0] for t in tiles]), d["vector_index"])
    assert np.array_equal(np.concatenate([t[1].ravel() for t in tiles]), d["nm_index"].astype(np.int64))
    assert np.array_equal(np.concatenate([t[2].ravel() for t in tiles]), d["kept_values"])
    assert np.array_equal(pack.vector_mask.cpu().numpy().astype(bool), d["vector_mask"])


@pytest.mark.parametrize("key", [k for k in NAMES if (k + "X") in Z.files])
def test_spmm_matches_reference(key):
    d = case(Z, key)
    enc = H.encode(d["W"], H.MaskPair(d["vector_mask"], d["element_mask"]),
                   H.GyroPermutation(d["sigma_o"], tuple(d["sigma_i"])), _cfg(d))
    pack = enc.device_pack()
    X = torch.as_tensor(d["X"].astype(np.float32)).cuda().to(torch.bfloat16).contiguous()
    ysimt = D.spmm_simt(pack, X).cpu().numpy().astype(np.float64)
    if _bf16_exact(d["W"]):
        assert O.relative_error(ysimt, d["Y"]) < 1e-5
    if D.spmm_supported(d["V"], d["N"], d["M"]) and _bf16_exact(d["W"]):
        Y = H.hinm_spmm(enc, d["X"])
        np.testing.assert_allclose(Y, d["Y"], rtol=RTOL, atol=ATOL)
        Yo = H.hinm_spmm_original_order(enc, d["X"])
        np.testing.assert_allclose(Yo, O.restore_row_order(d["Y"], d["sigma_o"]), rtol=RTOL, atol=ATOL)


def _tc_vs_simt(pack, B, seed, order="sigma"):
    X = torch.as_tensor(synth.randn_bf16((pack.n, B), seed)).cuda().to(torch.bfloat16)
    Y = D.spmm(pack, X, order=order).float()
    Yr = D.spmm_simt(pack, X, order=order)
    torch.cuda.synchronize()
    err = (Y - Yr).abs() - (ATOL + RTOL * Yr.abs())
    assert float(err.max()) <= 0, f"max excess {float(err.max())}"
    return Y, Yr


@pytest.mark.parametrize("V", [32, 64, 128])
@pytest.mark.parametrize("B", [8, 136, 520])
def test_spmm_tc_vs_simt_ragged_tokens(V, B):
    m, n = 4 * V, 768
    W = torch.as_tensor(synth.randn_bf16((m, n), 11)).cuda().to(torch.bfloat16)
    so = synth.random_sigma_o(m, 12)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, 0.5), so)
    for order in ("sigma", "original"):
        _tc_vs_simt(pack, B, 13, order)


def test_spmm_empty_tile_writes_zero_rows():
    V, m, n = 64, 256, 512
    Wh = synth.randn_bf16((m, n), 21)
    Wh[:V] = 0.0                                   # tile 0 (identity sigma_o) has zero scores
    pack = H.compress(torch.as_tensor(Wh).cuda().to(torch.bfloat16), H.HiNMConfig(V, 2, 4, 0.5),
                      np.arange(m))
    tp = pack.tile_ptr.cpu().numpy()
    assert tp[1] - tp[0] == 0, "global budget must starve the all-zero tile"
    X = torch.as_tensor(synth.randn_bf16((n, 64), 22)).cuda().to(torch.bfloat16)
    Y = torch.full((m, 64), 7.0, dtype=torch.bfloat16, device="cuda")
    D.spmm(pack, X, out=Y)
    torch.cuda.synchronize()
    assert float(Y[:V].abs().max()) == 0.0
    _tc_vs_simt(pack, 64, 22)


def test_cfg1_gyro_sigma():
    z = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    W = torch.as_tensor(synth.randn_bf16((768, 3072), 0)).cuda().to(torch.bfloat16)
    ptr = z["sigma_i_ptr"]
    si = [z["sigma_i"][ptr[t]:ptr[t + 1]].astype(np.int64) for t in range(12)]
    pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), z["sigma_o"].astype(np.int64), sigma_i=si)
    tiles = pack.to_host_tiles()
    assert np.array_equal(np.concatenate([t[0] for t in tiles]), z["vector_index"].astype(np.int64))
    assert np.array_equal(np.concatenate([t[1].ravel() for t in tiles]), z["nm_index"].astype(np.int64))
    X = torch.as_tensor(synth.randn_bf16((3072, 512), 1)).cuda().to(torch.bfloat16)
    Y = D.spmm(pack, X).float().cpu().numpy()
    np.testing.assert_allclose(Y, z["Y"].astype(np.float64), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("name", ["llama_down", "llama_up"])
def test_llama_shapes_bit_exact_and_spmm(name):
    spec = json.load(open(os.path.join(GOLDEN, "large.json")))[name]
    m, n = spec["m"], spec["n"]
    Wh = synth.randn_bf16((m, n), spec["w_seed"])
    W = torch.as_tensor(Wh).cuda().to(torch.bfloat16)
    so = synth.random_sigma_o(m, spec["sigma_o_seed"])
    cfg = H.HiNMConfig(64, 2, 4, 0.5)
    base = H.compress(W, cfg, so)                           # ascending survivors
    counts = np.diff(base.tile_ptr.cpu().numpy())
    assert counts.tolist() == spec["counts"]
    surv = [t[0] for t in base.to_host_tiles()]
    si = synth.permute_survivors(surv, spec["sigma_i_seed"])
    pack = H.compress(W, cfg, so, sigma_i=si)
    vidx = pack.vec_idx.cpu().numpy().astype("<i4")
    nmi = pack.nm_pos.cpu().numpy().astype(np.uint8)
    assert hashlib.sha256(vidx.tobytes()).hexdigest() == spec["vector_index_int32_sha256"]
    assert hashlib.sha256(nmi.tobytes()).hexdigest() == spec["nm_index_u8_sha256"]
    ys = np.load(os.path.join(GOLDEN, "large_y.npz"))[name].astype(np.float64)
    X = torch.as_tensor(synth.randn_bf16((n, 16), spec["x_seed"])).cuda().to(torch.bfloat16)
    Y = D.spmm(pack, X).float().cpu().numpy()
    np.testing.assert_allclose(Y, ys, rtol=RTOL, atol=ATOL)
    # full-size property check: tcgen05 == CUDA-core product over many token blocks
    _tc_vs_simt(pack, 2048, 5, "original")


def test_errors_follow_reference():
    cfg = H.HiNMConfig(4, 2, 4, 0.5)
    W = synth.randn_bf16((8, 16), 3).astype(np.float64)
    S = H.magnitude_saliency(W)
    vm = H.vector_prune(S, cfg, np.arange(8))
    surv = H.survivors_per_tile(vm)
    bad = list(surv)
    bad[1] = np.array(sorted(set(range(16)) - set(surv[1].tolist()))[: surv[1].size])
    with pytest.raises(H.InvariantViolation):
        H.nm_prune(S, vm, cfg, H.GyroPermutation(np.arange(8), tuple(bad)))
    # k_t % M != 0 with a matching sigma_i -> GroupingError (pruning.py:201-204); the
    # reference test at test_pruning.py:205-211 is known-bad (DimensionError fires first)
    cfg1 = H.HiNMConfig(1, 2, 4, 0.5)
    vm1 = np.zeros((2, 8), bool)
    vm1[0, :6] = True
    vm1[1, :2] = True
    with pytest.raises(H.GroupingError):
        H.nm_prune(np.ones((2, 8)), vm1, cfg1,
                   H.GyroPermutation(np.arange(2), (np.arange(6), np.arange(2))))
    # encode with an element kept inside a pruned vector (test_pruning.py:239-246)
    cfg2 = H.HiNMConfig(2, 1, 2, 0.5)
    W2 = synth.randn_bf16((4, 4), 4).astype(np.float64)
    S2 = H.magnitude_saliency(W2)
    vm2 = H.vector_prune(S2, cfg2, np.arange(4))
    sig2 = H.GyroPermutation(np.arange(4), tuple(H.survivors_per_tile(vm2)))
    em2 = H.nm_prune(S2, vm2, cfg2, sig2)
    em_bad = em2.copy()
    em_bad[0] = True
    with pytest.raises(H.InvariantViolation):
        H.encode(W2, H.MaskPair(vm2, em_bad), sig2, cfg2)
    enc = H.encode(W2, H.MaskPair(vm2, em2), sig2, cfg2)
    with pytest.raises(H.ShapeMismatch):
        H.hinm_spmm(enc, np.ones((5, 8)))


def test_compress_rejects_bad_sigma_i():
    V, m, n = 64, 128, 256
    W = torch.as_tensor(synth.randn_bf16((m, n), 31)).cuda().to(torch.bfloat16)
    cfg = H.HiNMConfig(V, 2, 4, 0.5)
    base = H.compress(W, cfg, np.arange(m))
    si = [t[0].copy() for t in base.to_host_tiles()]
    si[0][0] = si[0][1]                                    # duplicate column
    with pytest.raises(H.InvariantViolation):
        H.compress(W, cfg, np.arange(m), sigma_i=si)
