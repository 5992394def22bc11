"""GPU parity of the bytes the tcgen05 SpMM actually reads, and of the external-saliency compressor.

1. Operand image (north star: "vector indices, permutations and 2:4 metadata must be bit-exact"):
   the fused compressor's gidx / a_vals (UMMA K-major core matrices) / a_meta (tcgen05 2:4 E
   layout) are decoded back to vector_index / nm_index / kept_values twice -- by the C ABI
   (hinm_unpack_to_reference, OPERAND_IMAGE) and by an independent numpy decoder written here from
   the documented layout -- and compared bit-exactly with the reference's own encodings (goldens
   produced by running the reference: small.npz 2:4 cases with V in {32, 64, 128}, cfg1.npz with
   the reference gyro sigma, and the LLaMA-7B FFN SHA-256 digests of large.json).
2. External saliency (the reference's `encode --saliency` chain, cli.py:63-69,185-194): the GPU
   compressor and the drop-in vector_prune / nm_prune against reference outputs for positive,
   negative, fp32-valued and tie-heavy score matrices (tests/golden/make_golden_saliency.py).
"""

import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import GOLDEN, case, load_small  # noqa: E402

import paper_2407_20496_b200 as H  # noqa: E402
from paper_2407_20496_b200 import device as D  # noqa: E402
from paper_2407_20496_b200 import synth  # noqa: E402

Z, NAMES = load_small()
IMAGE_CASES = [k for k in NAMES if tuple(int(x) for x in Z[k + "meta"])[2:5] in
               ((32, 2, 4), (64, 2, 4), (128, 2, 4))]
RTOL, ATOL = 1e-2, 1e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def numpy_decode_image(pack):
    """Independent decoder of the operand image: -> (vec_idx, nm_pos, kept bits)."""
    V, T = pack.V, pack.T
    tp = pack.tile_ptr.cpu().numpy().astype(np.int64)
    kofs = pack.tile_kofs.cpu().numpy().astype(np.int64)
    eofs = pack.tile_eofs.cpu().numpy().astype(np.int64)
    gidx = pack.gidx.cpu().numpy()[:kofs[-1]]
    av = pack.a_vals.view(torch.int16).cpu().numpy().view(np.uint16)
    am = pack.a_meta.cpu().numpy().view(np.uint32)
    vi, nm, kv = [], [], []
    for t in range(T):
        k, kp = int(tp[t + 1] - tp[t]), int(kofs[t + 1] - kofs[t])
        G = k // 4
        assert kp == -(-k // 64) * 64
        g = gidx[kofs[t]:kofs[t] + kp]
        vi.append(g[:k])
        if k:
            assert np.all(g[k:] == g[k - 1]), "gather padding repeats the last real index"
        if G == 0:
            continue
        r = np.arange(V)[:, None]
        grp = np.arange(G)[None, :]
        # metadata: lane m0 + 8*k1 + 16*m2, word w, bits 16*m1 + 4*c of group 32e + 8w + 4k1 + c
        e, w, k1, c = grp >> 5, (grp >> 3) & 3, (grp >> 2) & 1, grp & 3
        m0, m1, m2 = r & 7, (r >> 3) & 1, r >> 4
        word = am[(eofs[t] + e) * V * 4 + (m0 + 8 * k1 + 16 * m2) * 4 + w]
        nib = (word >> (16 * m1 + 4 * c)) & 0xF
        pos = np.stack([nib & 3, nib >> 2], axis=-1)                     # (V, G, 2)
        assert np.all(pos[..., 0] < pos[..., 1])
        # values: compressed column cc = 2g + s; step cc // 16, core matrix (r/8, (cc%16)/8)
        cc = 2 * grp[..., None] + np.arange(2)[None, None, :]
        r3 = r[..., None]
        off = (kofs[t] // 2 * V + (cc >> 4) * 16 * V + (r3 >> 3) * 128 + ((cc & 15) >> 3) * 64
               + (r3 & 7) * 8 + (cc & 7))
        nm.append(pos.reshape(-1))
        kv.append(av[off].reshape(-1))
    cat = lambda a, dt: np.concatenate(a).astype(dt) if a else np.empty(0, dt)  # noqa: E731
    return cat(vi, np.int64), cat(nm, np.int64), cat(kv, np.uint16)


def _bits(x):
    return synth.bf16_bits(np.asarray(x, dtype=np.float32))


def _check_image(pack, vector_index, nm_index, kept_values):
    vi, nm, kv = numpy_decode_image(pack)
    assert np.array_equal(vi, np.asarray(vector_index, np.int64)), "gidx vs vector_index"
    assert np.array_equal(nm, np.asarray(nm_index, np.int64)), "a_meta vs nm_index"
    assert np.array_equal(kv, _bits(kept_values)), "a_vals vs kept_values"
    tp, vi2, nm2, kv2, so = pack.to_host_arrays("image")           # the C-ABI decoder
    assert np.array_equal(vi2, vi) and np.array_equal(nm2, nm)
    assert np.array_equal(_bits(kv2), kv)


@pytest.mark.parametrize("key", IMAGE_CASES)
def test_operand_image_decodes_to_reference_small(key):
    d = case(Z, key)
    W = torch.as_tensor(d["W"].astype(np.float32)).cuda().to(torch.bfloat16)
    from fractions import Fraction
    cfg = H.HiNMConfig(d["V"], 2, 4, Fraction(*d["s_v"]))
    pack = H.compress(W, cfg, d["sigma_o"], sigma_i=d["sigma_i"])
    _check_image(pack, d["vector_index"], d["nm_index"], d["kept_values"])
    # the image built from a host HiNMEncoding (hinm_pack_build) decodes identically
    enc = H.encode(d["W"], H.MaskPair(d["vector_mask"], d["element_mask"]),
                   H.GyroPermutation(d["sigma_o"], tuple(d["sigma_i"])), cfg)
    _check_image(enc.device_pack(), d["vector_index"], d["nm_index"], d["kept_values"])


def test_operand_image_decodes_to_reference_cfg1():
    z = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    W = torch.as_tensor(synth.randn_bf16((768, 3072), 0)).cuda().to(torch.bfloat16)
    ptr = z["sigma_i_ptr"]
    si = [z["sigma_i"][ptr[t]:ptr[t + 1]].astype(np.int64) for t in range(12)]
    pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), z["sigma_o"].astype(np.int64), sigma_i=si)
    vi, nm, kv = numpy_decode_image(pack)
    assert np.array_equal(vi, z["vector_index"].astype(np.int64))
    assert np.array_equal(nm, z["nm_index"].astype(np.int64))
    tiles = pack.to_host_tiles("image")
    assert np.array_equal(np.concatenate([t[1].ravel() for t in tiles]), z["nm_index"].astype(np.int64))


@pytest.mark.parametrize("name", ["llama_down", "llama_up"])
def test_operand_image_llama_digests(name):
    spec = json.load(open(os.path.join(GOLDEN, "large.json")))[name]
    m, n = spec["m"], spec["n"]
    W = torch.as_tensor(synth.randn_bf16((m, n), spec["w_seed"])).cuda().to(torch.bfloat16)
    so = synth.random_sigma_o(m, spec["sigma_o_seed"])
    cfg = H.HiNMConfig(64, 2, 4, 0.5)
    surv = [t[0] for t in H.compress(W, cfg, so).to_host_tiles()]
    pack = H.compress(W, cfg, so, sigma_i=synth.permute_survivors(surv, spec["sigma_i_seed"]))
    vi, nm, kv = numpy_decode_image(pack)
    assert hashlib.sha256(vi.astype("<i4").tobytes()).hexdigest() == spec["vector_index_int32_sha256"]
    assert hashlib.sha256(nm.astype(np.uint8).tobytes()).hexdigest() == spec["nm_index_u8_sha256"]
    # kept values: the image equals W at the decoded (row, column) positions
    tp = pack.tile_ptr.cpu().numpy()
    Wh = W.view(torch.int16).cpu().numpy().view(np.uint16)
    V = 64
    for t in (0, len(tp) // 2, len(tp) - 2):
        k = int(tp[t + 1] - tp[t])
        G = k // 4
        b = V * (int(tp[t]) // 4) * 2
        cols = vi[tp[t]:tp[t + 1]].reshape(G, 4)
        pos = nm[b:b + V * G * 2].reshape(V, G, 2)
        rows = so[t * V:(t + 1) * V]
        want = Wh[rows[:, None, None], cols[np.arange(G)[None, :, None], pos]]
        assert np.array_equal(kv[b:b + V * G * 2].reshape(V, G, 2), want)
    tp2, vi2, nm2, kv2, _ = pack.to_host_arrays("image")
    assert np.array_equal(vi2, vi) and np.array_equal(nm2, nm) and np.array_equal(_bits(kv2), kv)


def test_unpack_rejects_a_corrupted_image():
    W = torch.as_tensor(synth.randn_bf16((128, 256), 9)).cuda().to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), synth.random_sigma_o(128, 9))
    pack.to_host_arrays("image")
    bad = pack.a_meta.clone()
    bad[0] = 0x1B1B1B1B            # nibble 0xB: positions (3, 2) -- not ascending
    good, pack.a_meta = pack.a_meta, bad
    with pytest.raises(H.InvariantViolation):
        pack.to_host_arrays("image")
    pack.a_meta = good
    g = pack.gidx.clone()
    g[0] = 10 ** 6
    pack.gidx = g
    with pytest.raises(IndexError):
        pack.to_host_arrays("image")


# ------------------------------------------------------------------------------ external saliency
SZ = np.load(os.path.join(GOLDEN, "saliency.npz"))
SNAMES = [str(s) for s in SZ["names"]]


def _saliency_inputs(i):
    """Regenerates the inputs of tests/golden/make_golden_saliency.py (same seeds / streams)."""
    m, n, V, sv100, seed = (int(x) for x in SZ["cases"][i])
    kind = str(SZ["kinds"][i])
    rng = np.random.default_rng(1000 + seed)
    if kind == "abs_normal":
        S = np.abs(rng.standard_normal((m, n)))
    elif kind == "normal":
        S = rng.standard_normal((m, n))
    elif kind == "normal_f32":
        S = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64)
    else:
        S = rng.integers(-3, 4, size=(m, n)).astype(np.float64)
    W = synth.randn_bf16((m, n), 10 * seed).astype(np.float64)
    so = synth.random_sigma_o(m, 10 * seed + 1)
    X = synth.randn_bf16((n, 24), 10 * seed + 3).astype(np.float64)
    return m, n, V, sv100 / 100, seed, W, S, so, X


@pytest.mark.parametrize("i", range(len(SNAMES)), ids=SNAMES)
def test_compress_with_external_saliency_matches_reference(i):
    m, n, V, sv, seed, W, S, so, X = _saliency_inputs(i)
    p = SNAMES[i] + "_"
    cfg = H.HiNMConfig(V, 2, 4, sv)
    # the drop-in API with the same scores
    vm = H.vector_prune(S, cfg, so)
    assert np.array_equal(vm, SZ[p + "vector_mask"])
    si = synth.permute_survivors(H.survivors_per_tile(vm), 10 * seed + 2)
    em = H.nm_prune(S, vm, cfg, H.GyroPermutation(so, tuple(si)))
    assert np.array_equal(em, SZ[p + "element_mask"])
    # the fused device compressor with saliency (fp64 and, for fp32-valued scores, an fp32 tensor)
    Wd = torch.as_tensor(W.astype(np.float32)).cuda().to(torch.bfloat16)
    sal = torch.as_tensor(S).cuda()
    if SZ["kinds"][i] == "normal_f32":
        sal = sal.float()
    pack = H.compress(Wd, cfg, so, sigma_i=si, saliency=sal)
    assert np.array_equal(pack.vector_mask.cpu().numpy().astype(bool), SZ[p + "vector_mask"])
    tiles = pack.to_host_tiles()
    assert np.array_equal(np.concatenate([t[0] for t in tiles]), SZ[p + "vector_index"])
    assert np.array_equal(np.concatenate([t[1].ravel() for t in tiles]), SZ[p + "nm_index"].astype(np.int64))
    assert np.array_equal(np.concatenate([t[2].ravel() for t in tiles]), SZ[p + "kept_values"])
    _check_image(pack, SZ[p + "vector_index"], SZ[p + "nm_index"], SZ[p + "kept_values"])
    Y = D.spmm(pack, torch.as_tensor(X.astype(np.float32)).cuda().to(torch.bfloat16)).float().cpu().numpy()
    np.testing.assert_allclose(Y, SZ[p + "Y"], rtol=RTOL, atol=ATOL)


def test_saliency_rejects_non_finite():
    W = torch.as_tensor(synth.randn_bf16((128, 256), 1)).cuda().to(torch.bfloat16)
    S = np.ones((128, 256))
    S[3, 4] = np.nan
    with pytest.raises(ValueError):
        H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.arange(128), saliency=S)
    with pytest.raises(ValueError):
        H.vector_prune(S, H.HiNMConfig(64, 2, 4, 0.5), np.arange(128))


def test_sigma_o_out_of_range_raises_index_error():
    W = torch.as_tensor(synth.randn_bf16((128, 256), 1)).cuda().to(torch.bfloat16)
    so = np.arange(128)
    so[5] = 128
    with pytest.raises(IndexError):
        H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), so)
    with pytest.raises(IndexError):
        H.vector_prune(np.abs(W.float().cpu().numpy()), H.HiNMConfig(64, 2, 4, 0.5), so)
    with pytest.raises(H.ShapeMismatch):
        H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.arange(64))


def test_spmm_checks_out_and_device():
    W = torch.as_tensor(synth.randn_bf16((128, 256), 1)).cuda().to(torch.bfloat16)
    pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), np.arange(128))
    X = torch.zeros(256, 16, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        D.spmm(pack, X, out=torch.empty(128, 16, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        D.spmm(pack, X, out=torch.empty(128, 8, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):
        D.spmm(pack, X, order="backwards")
