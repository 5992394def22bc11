"""GPU parity of the union-group image (csrc/group.cu) and the CTA-pair SpMM (spmm_sm100.cu PAIR).

The union-group image is a B200 layout of the same HiNMEncoding: 256 // V consecutive tiles share
one gather list.  Parity is checked two ways:
  * bit-exact: the image the MMA reads (gidx, a_vals, a_meta of the pseudo pack, decoded by
    hinm_unpack_to_reference) maps back, row by row, to exactly the reference view's nonzero
    (column, value) pairs -- every kept value once, at its column, nothing else nonzero;
  * SpMM: Y from the CTA-pair kernel against the oracle (reference float64 product) at the
    north-star tolerance, rtol 1e-2 / atol 1e-3, in sigma_o and original row order, and equal to the
    per-tile image's Y up to fp32 summation order.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hinm_oracle as O  # noqa: E402

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402

RTOL, ATOL = 1e-2, 1e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _pack(m, n, V, sv=0.5, seed=0, zero_tiles=()):
    W = synth.randn_bf16((m, n), seed)
    for t in zero_tiles:  # a tile that loses every vector still sits in its group
        W[t * V:(t + 1) * V] = 0.0
    so = synth.random_sigma_o(m, seed + 1)
    cfg = H.HiNMConfig(V, 2, 4, sv)
    Wd = torch.as_tensor(W.astype(np.float32)).cuda().to(torch.bfloat16)
    return W, so, cfg, H.compress(Wd, cfg, so, groups=True)


def _row_maps_reference(pack):
    """{(tile, row): {column: value bits}} of the reference view (nonzero kept values)."""
    out = {}
    for t, (vi, nm, kv) in enumerate(pack.to_host_tiles()):
        for r in range(pack.V):
            d = {}
            for g in range(nm.shape[1] // 2):
                for j in range(2):
                    v = kv[r, 2 * g + j]
                    if v != 0.0:
                        d[int(vi[4 * g + nm[r, 2 * g + j]])] = v
            out[(t, r)] = d
    return out


def _row_maps_group(pack, source):
    """The same maps decoded from the union-group pseudo pack (its operand image or view)."""
    g = pack.group
    Gt = 256 // pack.V
    out = {}
    for tp, (vi, nm, kv) in enumerate(g.to_host_tiles(source)):
        u, h = divmod(tp, 2)
        for r2 in range(128):
            R = h * 128 + r2
            t, rl = u * Gt + R // pack.V, R % pack.V
            d = {}
            for c in range(nm.shape[1] // 2):
                for j in range(2):
                    v = kv[r2, 2 * c + j]
                    if v != 0.0:
                        col = int(vi[4 * c + nm[r2, 2 * c + j]])
                        assert col not in d, f"column {col} twice in row {R} of group {u}"
                        d[col] = v
            if t >= pack.T:
                assert not d, f"padding row {R} of group {u} has nonzeros"
                continue
            out[(t, rl)] = d
    return out


CASES = [  # (m, n, V, s_v)
    (512, 1024, 64, 0.5),
    (512, 768, 32, 0.5),
    (256, 2048, 64, 0.75),
    (320, 512, 64, 0.5),     # partial last group (64 real rows of 256)
    (192, 512, 32, 0.5),     # one partial group
    (1024, 4096, 64, 0.5),   # LLaMA-like n
]


@pytest.mark.parametrize("m,n,V,sv", CASES)
def test_group_image_bit_exact(m, n, V, sv):
    _, _, _, pack = _pack(m, n, V, sv)
    assert pack.group is not None and pack.group.pair == 1 and pack.group.rows == m
    ref = _row_maps_reference(pack)
    for source in ("view", "image"):
        got = _row_maps_group(pack, source)
        assert got.keys() == ref.keys()
        for key in ref:
            assert got[key] == ref[key], f"{source}: row {key} differs"


def test_group_image_empty_tile():
    _, _, _, pack = _pack(512, 1024, 64, 0.5, seed=3, zero_tiles=(1,))
    ref = _row_maps_reference(pack)
    got = _row_maps_group(pack, "image")
    assert got == ref


def test_group_plan_deterministic():
    _, _, _, pack = _pack(512, 2048, 64, 0.5, seed=5)
    a = pack.group.to_host_arrays("image")
    H.build_group_image(pack)
    b = pack.group.to_host_arrays("image")
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("m,n,V,sv", CASES)
@pytest.mark.parametrize("B", [256, 520])
def test_pair_spmm_matches_oracle(m, n, V, sv, B):
    W, so, cfg, pack = _pack(m, n, V, sv, seed=11)
    Xh = synth.randn_bf16((n, B), 12)
    X = torch.as_tensor(Xh.astype(np.float32)).cuda().to(torch.bfloat16)
    tiles = pack.to_host_tiles()
    Yref = O.hinm_spmm(tiles, Xh.astype(np.float64), m, V, 2, 4)
    for order, ref in (("sigma", Yref), ("original", O.restore_row_order(Yref, so))):
        Yg = H.spmm(pack, X, order=order, image="groups").float().cpu().numpy()
        np.testing.assert_allclose(Yg, ref, rtol=RTOL, atol=ATOL)
        Yt = H.spmm(pack, X, order=order, image="tiles").float().cpu().numpy()
        np.testing.assert_allclose(Yg, Yt, rtol=1e-2, atol=1e-2)


def test_pair_spmm_llama_shapes_sampled():
    """LLaMA-7B FFN shapes at the bench's token count (sampled token columns vs the oracle)."""
    for (m, n) in ((11008, 4096), (4096, 11008)):
        W, so, cfg, pack = _pack(m, n, 64, 0.5, seed=21)
        B = 2048
        Xh = synth.randn_bf16((n, B), 22)
        X = torch.as_tensor(Xh.astype(np.float32)).cuda().to(torch.bfloat16)
        Y = H.spmm(pack, X, order="original", image="groups").float().cpu().numpy()
        cols = np.arange(0, B, 97)
        ref = O.restore_row_order(O.hinm_spmm(pack.to_host_tiles(), Xh[:, cols].astype(np.float64), m, 64, 2, 4), so)
        np.testing.assert_allclose(Y[:, cols], ref, rtol=RTOL, atol=ATOL)


def test_auto_picks_images_by_token_count():
    """The per-call choice: the union-group image at LLaMA scale, the per-tile image where the
    pairs would idle (a 768-row layer at 256 tokens: 3 groups vs 12 tiles)."""
    from paper_2407_20496_b200 import _lib

    lib = _lib.load()
    _, _, _, pack = _pack(11008, 4096, 64, 0.5, seed=31)
    X = torch.zeros(4096, 16384, dtype=torch.bfloat16, device="cuda")
    H.spmm(pack, X)
    assert lib.hinm_last_launch_count() == 1 and lib.hinm_last_image() == 1
    H.spmm(pack, X, image="tiles")
    assert lib.hinm_last_image() == 0
    _, _, _, small = _pack(768, 768, 64, 0.5, seed=32)
    H.spmm(small, torch.zeros(768, 256, dtype=torch.bfloat16, device="cuda"))
    assert lib.hinm_last_image() == 0


def test_replicate_keeps_group():
    _, _, _, pack = _pack(512, 1024, 64, 0.5, seed=41)
    rep = pack.replicate("cuda:0")
    assert rep.group is not None and rep.group.pair == 1
    X = torch.as_tensor(synth.randn_bf16((1024, 256), 42).astype(np.float32)).cuda().to(torch.bfloat16)
    a = H.spmm(pack, X, image="groups")
    b = H.spmm(rep, X, image="groups")
    assert torch.equal(a, b)


def test_early_weight_streams_after_pack_writers():
    """Short SpMM launches (PDL) stream their weights before griddepcontrol.wait; every pack writer
    ends with hinm_stream_fence.  Back-to-back compress -> spmm, rebuild -> spmm and replicate ->
    spmm sequences on one stream, with the weights changing every iteration, must match the
    CUDA-core kernel (which reads the reference view, after a synchronize)."""
    X = torch.as_tensor(synth.randn_bf16((512, 264), 51).astype(np.float32)).cuda().to(torch.bfloat16)
    for i in range(6):
        W = torch.as_tensor(synth.randn_bf16((512, 512), 60 + i).astype(np.float32)).cuda().to(torch.bfloat16)
        so = synth.random_sigma_o(512, 70 + i)
        pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), so, groups=True)
        outs = [H.spmm(pack, X, order="original", image=img) for img in ("tiles", "groups")]
        H.build_group_image(pack)
        outs.append(H.spmm(pack, X, order="original", image="groups"))
        rep = pack.replicate("cuda:0")
        outs.append(H.spmm(rep, X, order="original", image="groups"))
        torch.cuda.synchronize()
        ref = H.spmm_simt(pack, X, order="original")
        for Y in outs:
            err = (Y.float() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
            assert err < 1e-2, (i, err)
