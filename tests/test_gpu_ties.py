"""GPU parity on tie-heavy weights at a size that takes the multi-CTA budget select (T x G > 16384).

Few distinct |W| values make many column scores and group gains equal, so the rank's histogram
bin holds thousands of keys: with all magnitudes equal every gain is tied and the threshold pick
takes its radix fallback (more candidates than the candidate list holds), and the per-tile counts
come from the (q, t) tie order alone (pruning.py:115-128: the greedy takes the earlier chunk, then
the lower tile).  Also the tile sort's tie handling (equal scores -> lower column first) and the
2:4 select's ties (equal magnitudes -> lower position).  Everything bit-exact against the oracle.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hinm_oracle as O  # noqa: E402

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _weights(kind, m, n, seed, so, V):
    """Tie-heavy magnitudes, scaled per tile by 4 / 2 / 1 (t mod 3) so that tiles of one class tie
    with each other and the budget's threshold falls inside the middle class."""
    rng = np.random.default_rng(seed)
    sign = np.where(rng.random((m, n)) < 0.5, -1.0, 1.0)
    if kind == "all_equal":      # every score, gain and 2:4 candidate tied
        mag = np.ones((m, n))
    elif kind == "two_values":   # |W| in {1, 2}: ~65 distinct scores, hundreds of equal gains each
        mag = np.where(rng.random((m, n)) < 0.5, 1.0, 2.0)
    else:                        # a tied block: the first half of the columns equal, the rest random
        mag = np.abs(synth.randn_bf16((m, n), seed).astype(np.float64))
        mag[:, : n // 2] = 0.5
    fac = np.empty(m)
    for t in range(m // V):
        fac[so[t * V:(t + 1) * V]] = (4.0, 2.0, 1.0)[t % 3]
    return (sign * mag * fac[:, None]).astype(np.float64)


@pytest.mark.parametrize("kind", ["all_equal", "two_values", "half_tied"])
@pytest.mark.parametrize("V", [64, 32])
def test_tie_heavy_compress_bit_exact(kind, V):
    from fractions import Fraction

    m, n = 2048, 4096
    so = synth.random_sigma_o(m, 3)
    Wd = _weights(kind, m, n, 7, so, V)
    assert np.array_equal(synth.bf16_round(Wd.astype(np.float32)).astype(np.float64), Wd)
    assert (m // V) * (n // 4) > 16384  # the multi-CTA budget select
    W = torch.as_tensor(Wd.astype(np.float32)).cuda().to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(V, 2, 4, Fraction(5, 8)), so)
    ref = O.compress(Wd, so, V, 2, 4, pack.total_keep)
    assert np.array_equal(np.diff(pack.tile_ptr.cpu().numpy()), ref["counts"])
    got = pack.to_host_tiles()
    assert len(got) == len(ref["tiles"])
    for t, ((gv, gn, gk), (rv, rn, rk)) in enumerate(zip(got, ref["tiles"])):
        assert np.array_equal(gv, rv), f"tile {t}: vector_index"
        assert np.array_equal(gn, rn), f"tile {t}: nm_index"
        assert np.array_equal(gk, rk), f"tile {t}: kept values"
