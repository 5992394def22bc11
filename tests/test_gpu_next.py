"""GPU: §8(f) rows 2-4 -- file formats driving the device pack, multi-layer chains without
restore, and group-order freedom -- against the reference's own outputs
(tests/golden/next.npz, tests/golden/io/, tests/golden/make_golden_next.py) and the oracle."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hinm_oracle as O  # noqa: E402  (test infrastructure)
import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import io as hio  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402
from paper_2407_20496_b200.model import GyroPermutation, MaskPair  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CFG = H.HiNMConfig(64, 2, 4, 0.5)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture(scope="module")
def nxt():
    return np.load(os.path.join(GOLD, "next.npz"))


def test_build_layer_chain_matches_reference(nxt):
    chain = H.build_layer_chain([nxt["chain_W1"], nxt["chain_W2"]], CFG, permute=H.no_perm_prune)
    for l, enc in enumerate(chain.layers):
        assert np.array_equal(enc.sigma_o, nxt[f"chain_l{l}_sigma_o"])
        for t, tile in enumerate(enc.tiles):
            assert np.array_equal(tile.vector_index, nxt[f"chain_l{l}_t{t}_vi"])
            assert np.array_equal(tile.nm_index, nxt[f"chain_l{l}_t{t}_nm"])
            assert np.array_equal(tile.kept_values, nxt[f"chain_l{l}_t{t}_kv"])


def test_build_layer_chain_default_gyro_matches_reference():
    """The reference's own build_layer_chain with its default search (gyro_permute, reduced budgets):
    identical sigma_o, encodings and chain output (tests/golden/make_golden_chain.py)."""
    z = np.load(os.path.join(GOLD, "chain_gyro.npz"))
    cfg = H.HiNMConfig(vector_size=32, nm_keep=2, nm_group=4, vector_sparsity=0.5, ocp_max_iters=3,
                       icp_max_iters=3, seed=5)
    W1 = synth.randn_bf16((128, 96), 51).astype(np.float64)
    W2 = synth.randn_bf16((64, 128), 52).astype(np.float64)
    X = synth.randn_bf16((96, 16), 53).astype(np.float64)
    chain = H.build_layer_chain([W1, W2], cfg)
    for l, enc in enumerate(chain.layers):
        assert np.array_equal(enc.sigma_o, z[f"l{l}_sigma_o"])
        assert np.array_equal(np.concatenate([t.vector_index for t in enc.tiles]), z[f"l{l}_vi"])
        assert np.array_equal(np.concatenate([t.nm_index.ravel() for t in enc.tiles]), z[f"l{l}_nm"])
        assert np.array_equal(np.concatenate([t.kept_values.ravel() for t in enc.tiles]), z[f"l{l}_kv"])
    assert np.array_equal(chain.final_sigma_o, z["final_sigma_o"])
    assert O.relative_error(H.compose_layers(chain, X), z["Y"]) < 1e-2


def test_compose_layers_matches_reference(nxt):
    chain = H.build_layer_chain([nxt["chain_W1"], nxt["chain_W2"]], CFG, permute=H.no_perm_prune)
    Y = H.compose_layers(chain, nxt["chain_X"])
    # two bf16 layers (bf16 activations between them, fp32 accumulation) vs float64
    assert O.relative_error(Y, nxt["chain_Y"]) < 1e-2


def _random_sigma_permute(seed):
    rng = np.random.default_rng(seed)

    def permute(W, cfg, saliency=None):
        m, _ = W.shape
        so = rng.permutation(m)
        S = np.abs(W) if saliency is None else saliency
        vm = H.vector_prune(S, cfg, so)
        sig = GyroPermutation(sigma_o=so, sigma_i=tuple(H.survivors_per_tile(vm)))
        return sig, MaskPair(vector_mask=vm, element_mask=H.nm_prune(S, vm, cfg, sig)), None
    return permute


def test_chain_without_restore_random_sigma():
    """Layer l's columns are pre-permuted by layer l-1's sigma_o, so no restore between layers:
    the chain equals the dense product of the decoded (sigma_o-ordered) layers."""
    Ws = [synth.randn_bf16((256, 192), 41).astype(np.float64),
          synth.randn_bf16((128, 256), 42).astype(np.float64),
          synth.randn_bf16((192, 128), 43).astype(np.float64)]
    X = synth.randn_bf16((192, 40), 44).astype(np.float64)
    chain = H.build_layer_chain(Ws, CFG, permute=_random_sigma_permute(5))
    assert not np.array_equal(chain.layers[0].sigma_o, np.arange(256))
    ref = X
    for enc in chain.layers:
        ref = H.decode(enc, enc.shape) @ ref
    Y = H.compose_layers(chain, X)
    assert Y.shape == (192, 40)
    assert O.relative_error(Y, ref) < 1e-2
    # CUDA-tensor inputs stay on the device
    Yd = H.compose_layers(chain, torch.as_tensor(X.astype(np.float32)).cuda())
    assert Yd.is_cuda and O.relative_error(Yd.float().cpu().numpy(), ref) < 1e-2


def test_tile_shuffle_check_passes():
    W = torch.as_tensor(synth.randn_bf16((256, 512), 51)).to("cuda", torch.bfloat16)
    pack = H.compress(W, CFG, synth.random_sigma_o(256, 52))
    enc = H.encoding_from_pack(pack)
    X = synth.randn_bf16((512, 64), 53).astype(np.float64)
    rep = H.tile_shuffle_check(enc, X, np.random.default_rng(9), trials=3)
    assert rep["kept_sets_equal"] and rep["passed"], rep
    assert rep["max_relative_error"] < 1e-5
    assert rep["tc_max_relative_error"] < 1e-2


def test_pack_file_roundtrip(tmp_path):
    W = torch.as_tensor(synth.randn_bf16((384, 640), 61)).to("cuda", torch.bfloat16)
    pack = H.compress(W, CFG, synth.random_sigma_o(384, 62))
    hio.save_pack(pack, tmp_path / "enc.json")
    back = hio.load_pack(tmp_path / "enc.json")
    X = torch.as_tensor(synth.randn_bf16((640, 96), 63)).to("cuda", torch.bfloat16)
    y0 = H.spmm(pack, X, order="original")
    y1 = H.spmm(back, X, order="original")
    assert torch.equal(y0, y1)


def test_load_pack_from_reference_file():
    """The reference-written encoding JSON (V=4, CUDA-core kernel) drives the GPU product."""
    enc = hio.load_encoding(os.path.join(GOLD, "io", "encoding.json"))
    X = synth.randn_bf16((32, 16), 71).astype(np.float64)
    Y = H.hinm_spmm(enc, X)
    tiles = [(t.vector_index, t.nm_index, t.kept_values) for t in enc.tiles]
    ref = O.hinm_spmm(tiles, X, 16, 4, 2, 4)
    assert O.relative_error(Y, ref) < 1e-2
    pack = hio.load_pack(os.path.join(GOLD, "io", "encoding.json"))
    assert pack.m == 16 and pack.n == 32 and pack.T == 4
