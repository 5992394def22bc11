"""GPU: compress_layers (several weights on side streams at once) gives the same packs as one
compress per layer, bit-exact against the oracle's vector_prune -> nm_prune -> encode
(reference pruning.py:150-164,182-213,284-324), and its packs are usable on the caller's stream
without a host synchronisation."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hinm_oracle as O  # noqa: E402  (test infrastructure)
import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


FIELDS = ("sigma_o", "tile_ptr", "vec_idx", "nm_pos", "kept", "tile_kofs", "tile_eofs")


def _same(a, b):
    for f in FIELDS:
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    kp = int(a.tile_kofs[-1])
    assert torch.equal(a.gidx[:kp], b.gidx[:kp])
    assert torch.equal(a.a_vals[:kp * a.V // 2], b.a_vals[:kp * b.V // 2])


@pytest.mark.parametrize("streams", [1, 2, 3])
def test_compress_layers_equals_per_layer_compress(streams):
    shapes = [(256, 1024), (512, 768), (128, 2048), (384, 512)]
    cfgs = [H.HiNMConfig(64, 2, 4, 0.5), H.HiNMConfig(32, 2, 4, 0.75), H.HiNMConfig(128, 2, 4, 0.5),
            H.HiNMConfig(64, 2, 4, 0.5)]
    Ws = [torch.as_tensor(synth.randn_bf16(s, 10 + i)).to("cuda", torch.bfloat16)
          for i, s in enumerate(shapes)]
    sos = [synth.random_sigma_o(s[0], 20 + i) for i, s in enumerate(shapes)]
    # one sigma_o as a CUDA tensor (copied on the device), the others from the host
    sos_in = [torch.as_tensor(so).cuda() if i == 1 else so for i, so in enumerate(sos)]
    packs = H.compress_layers(Ws, cfgs, sos_in, groups=False, streams=streams)
    for W, c, so, p in zip(Ws, cfgs, sos, packs):
        _same(p, H.compress(W, c, so, groups=False))
    # bit-exact against the oracle for the first layer
    W0 = Ws[0].float().cpu().numpy().astype(np.float64)
    m, n = shapes[0]
    ref = O.compress(W0, sos[0], 64, 2, 4, (m // 64) * (n // 2))
    for (gv, gn, gk), (rv, rn, rk) in zip(packs[0].to_host_tiles(), ref["tiles"]):
        assert np.array_equal(gv, rv) and np.array_equal(gn, rn) and np.array_equal(gk, rk)


def test_compress_layers_packs_ready_on_caller_stream():
    """SpMM right after compress_layers on the caller's stream, no synchronize in between."""
    m, n, B = 256, 1024, 256
    cfg = H.HiNMConfig(64, 2, 4, 0.5)
    Wh = [synth.randn_bf16((m, n), 30 + i) for i in range(3)]
    so = [synth.random_sigma_o(m, 40 + i) for i in range(3)]
    Xh = synth.randn_bf16((n, B), 50)
    X = torch.as_tensor(Xh).to("cuda", torch.bfloat16)
    packs = H.compress_layers([torch.as_tensor(w).to("cuda", torch.bfloat16) for w in Wh], cfg, so)
    Ys = [H.spmm(p, X, order="original") for p in packs]
    torch.cuda.synchronize()
    for w, s, Y in zip(Wh, so, Ys):
        ref = O.compress(w.astype(np.float64), s, 64, 2, 4, (m // 64) * (n // 2))
        Yr = O.restore_row_order(O.hinm_spmm(ref["tiles"], Xh.astype(np.float64), m, 64, 2, 4), s)
        np.testing.assert_allclose(Y.float().cpu().numpy(), Yr, rtol=1e-2, atol=1e-3)


def test_compress_layers_argument_checks():
    W = torch.as_tensor(synth.randn_bf16((256, 512), 1)).to("cuda", torch.bfloat16)
    with pytest.raises(H.ShapeMismatch):
        H.compress_layers([W, W], H.HiNMConfig(64, 2, 4, 0.5), [np.arange(256)])
    assert H.compress_layers([], H.HiNMConfig(64, 2, 4, 0.5), []) == []
