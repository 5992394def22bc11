"""GPU: the exact step bench.py times, checked against the oracle (test infrastructure).

LLaMA-7B FFN at 75% HiNM (V=64, 2:4, s_v=0.5): gate and up (11008x4096) on X, down (4096x11008)
on the up projection's bf16 output, every SpMM with the sigma_o restore fused (ORIGINAL order),
at the bench's 16384 tokens, at 2048 (BASELINE cfg3's low end, = one rank of the 8-way shard of
16384) and at 256 (one rank of the 8-way shard of 2048, where the launcher switches to 128-token
units).  The packs are first checked bit-exactly against the oracle's compressor; then 64 sampled
token columns of every output are compared with the oracle's float64 hinm_spmm +
restore_row_order on the identical inputs (rtol 1e-2 / atol 1e-3, the north-star tolerance for bf16
inputs with fp32 accumulation).

Weights are N(0, 1/n) (the scale of a trained / initialised linear layer) so that outputs are O(1)
and the absolute part of the tolerance means what it says: with N(0, 1) weights the down projection's
outputs reach ~1e4 and single near-cancelling entries carry ~1e-2 of fp32 accumulation error --
below the reference's own relative_error bound (checked too) but not an atol of 1e-3.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hinm_oracle as O  # noqa: E402  (test infrastructure)

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402

RTOL, ATOL = 1e-2, 1e-3
V = 64
LAYERS = [("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture(scope="module")
def layers():
    cfg = H.HiNMConfig(V, 2, 4, 0.5)
    out = {}
    for i, (name, m, n) in enumerate(LAYERS):
        Wh = synth.bf16_round(synth.randn_bf16((m, n), 100 + i) / np.float32(np.sqrt(n)))
        so = synth.random_sigma_o(m, 200 + i)
        pack = H.compress(torch.as_tensor(Wh).cuda().to(torch.bfloat16), cfg, so)
        ref = O.compress(Wh.astype(np.float64), so, V, 2, 4, (m // V) * (n // 2))
        for (gv, gn, gk), (rv, rn, rk) in zip(pack.to_host_tiles(), ref["tiles"]):
            assert np.array_equal(gv, rv) and np.array_equal(gn, rn) and np.array_equal(gk, rk)
        out[name] = (pack, ref["tiles"], so, m)
    return out


@pytest.mark.parametrize("tokens", [16384, 2048, 256])
def test_bench_step_matches_oracle(layers, tokens):
    Xh = synth.randn_bf16((4096, tokens), 300 + tokens)
    X = torch.as_tensor(Xh).cuda().to(torch.bfloat16)
    y = {name: torch.empty(m, tokens, dtype=torch.bfloat16, device="cuda") for name, m, _ in LAYERS}
    p = {k: v[0] for k, v in layers.items()}
    # the bench step (bench.py run_llama.step)
    H.spmm(p["gate"], X, out=y["gate"], order="original")
    H.spmm(p["up"], X, out=y["up"], order="original")
    H.spmm(p["down"], y["up"], out=y["down"], order="original")
    torch.cuda.synchronize()
    cols = np.sort(np.random.default_rng(tokens).choice(tokens, size=min(64, tokens), replace=False))
    ci = torch.as_tensor(cols).cuda()
    xs = Xh.astype(np.float64)[:, cols]
    up_in = y["up"].index_select(1, ci).float().cpu().numpy().astype(np.float64)  # down's actual input
    for name, inp in (("gate", xs), ("up", xs), ("down", up_in)):
        _, tiles, so, m = layers[name]
        ref = O.restore_row_order(O.hinm_spmm(tiles, inp, m, V, 2, 4), so)
        got = y[name].index_select(1, ci).float().cpu().numpy().astype(np.float64)
        np.testing.assert_allclose(got, ref, rtol=RTOL, atol=ATOL, err_msg=f"{name} @ {tokens} tokens")
        assert O.relative_error(got, ref) < 1e-2
