"""Drop-in replacements for the reference's pruning / encoding API (pkg/src/hinm/pruning.py).

Same names, argument meaning, return types and exception classes as the reference; the
array work runs in libhinm_b200.so on the GPU:

  vector_prune  pruning.py:150-164  -> hinm_vector_prune  (scores, per-tile sort, budget)
  nm_prune      pruning.py:182-213  -> hinm_nm_select(SCORES)
  encode        pruning.py:284-324  -> hinm_nm_select(MASK) (+ validate_masks :226-254)
  decode / restore_row_order / apply_masks stay host utilities, as in the reference.

Inputs may be numpy arrays, DenseMatrix/SaliencyMatrix, or torch tensors (CPU or CUDA).
Host inputs are uploaded to the current CUDA device and results come back as numpy arrays;
CUDA tensor inputs keep results on the device where the reference returns arrays.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DeviceError, InvariantViolation, NegativeScore, ShapeMismatch
from .model import (DenseMatrix, GyroPermutation, HiNMConfig, MaskPair, SaliencyMatrix,
                    ValidatedConfig, as_values, ensure_validated)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the HiNM hot path runs only on the GPU (no CPU fallback)")
    return torch


def _is_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and x.is_cuda


def _dev_f64(x, torch):
    """fp64 CUDA tensor view of a matrix input."""
    if isinstance(x, DenseMatrix):
        x = x.values
    elif isinstance(x, SaliencyMatrix):
        x = x.scores
    if _is_cuda(x):
        return x.to(torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(as_values(x), dtype=np.float64)).cuda()


def _dev_i32(x, torch, device):
    if _is_cuda(x):
        return x.to(device=device, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.int64)).astype(np.int32)).to(device)


def check_sigma_o(sigma_o, m: int) -> None:
    """Host-side guard before any kernel indexes W with sigma_o: ShapeMismatch for a wrong
    length, IndexError for an entry outside [0, m) (the reference's fancy index ``S[rows]``,
    pruning.py:63-80, raises IndexError there).  CUDA tensors are checked with one reduction."""
    if _is_cuda(sigma_o):
        n = sigma_o.numel()
        lo = int(sigma_o.min()) if n else 0
        hi = int(sigma_o.max()) if n else -1
    else:
        a = np.asarray(sigma_o)
        if a.ndim != 1:
            raise ShapeMismatch(f"sigma_o must be 1-D, got shape {a.shape}")
        n = a.size
        lo = int(a.min()) if n else 0
        hi = int(a.max()) if n else -1
    if n != m:
        raise ShapeMismatch(f"sigma_o has {n} entries for {m} rows")
    if lo < 0 or hi >= m:
        raise IndexError(f"sigma_o entry {lo if lo < 0 else hi} out of range for {m} rows")


def _check_scores(saliency, S) -> None:
    """Raw score arrays may hold any real value (the reference sorts -score with lexsort, and the
    device keys are order-preserving for negatives); NaN / Inf have no reference order here and
    are rejected.  SaliencyMatrix inputs were already checked by their constructor."""
    if isinstance(saliency, SaliencyMatrix):
        return
    import torch

    if not bool(torch.isfinite(S).all()):
        raise ValueError("saliency contains NaN or infinite values")


def _sigma_csr(sigma_i, T, torch, device):
    sizes = [int(np.asarray(s).size) for s in sigma_i]
    if len(sizes) != T:
        raise InvariantViolation(f"sigma_i has {len(sizes)} tiles, expected {T}")
    ptr = np.zeros(T + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(sizes)
    flat = np.concatenate([np.asarray(s, dtype=np.int64).ravel() for s in sigma_i]) if T else \
        np.empty(0, np.int64)
    return (torch.as_tensor(ptr.astype(np.int32)).to(device),
            torch.as_tensor(flat.astype(np.int32) if flat.size else np.zeros(1, np.int32)).to(device),
            ptr)


def magnitude_saliency(weights) -> SaliencyMatrix:
    """|w| importance (pruning.py:37-39)."""
    if _is_cuda(weights):
        weights = weights.detach().float().cpu().numpy()
    return SaliencyMatrix(np.abs(as_values(weights)))


def tile_rows(sigma_o, vector_size: int) -> np.ndarray:
    """Original row ids per tile (pruning.py:63-65)."""
    return np.asarray(sigma_o, dtype=np.int64).reshape(-1, vector_size)


def survivors_per_tile(vector_mask) -> list[np.ndarray]:
    """Ascending surviving column ids per tile (pruning.py:167-169)."""
    vm = vector_mask.cpu().numpy() if hasattr(vector_mask, "cpu") else np.asarray(vector_mask)
    return [np.flatnonzero(row) for row in vm]


def vector_prune(saliency, cfg, sigma_o):
    """(T, n) boolean vector mask under output order sigma_o (pruning.py:150-164), on the GPU."""
    torch = _torch()
    on_device = _is_cuda(saliency)
    S = _dev_f64(saliency, torch)
    m, n = S.shape
    vcfg = ensure_validated(cfg, (m, n))
    dev = S.device
    _check_scores(saliency, S)
    check_sigma_o(sigma_o, m)
    so = _dev_i32(sigma_o, torch, dev)
    lib = _lib.load()
    wsb = ctypes.c_size_t()
    _lib.check(lib.hinm_compress_workspace(m, n, vcfg.vector_size, vcfg.nm_group,
                                           ctypes.byref(wsb)), "workspace")
    ws = torch.empty(max(wsb.value, 1), dtype=torch.uint8, device=dev)
    T = vcfg.num_tiles
    tile_ptr = torch.empty(T + 1, dtype=torch.int32, device=dev)
    surv = torch.empty(max(vcfg.total_keep, 1), dtype=torch.int32, device=dev)
    vmask = torch.empty(T, n, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = lib.hinm_vector_prune(None, 0, None, 0, S.data_ptr(), S.stride(0), so.data_ptr(), m, n,
                                   vcfg.vector_size, vcfg.nm_group, vcfg.total_keep,
                                   tile_ptr.data_ptr(), surv.data_ptr(), vmask.data_ptr(),
                                   ws.data_ptr(), wsb.value, torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "vector_prune")
    out = vmask.bool()
    return out if on_device else out.cpu().numpy()


def nm_prune(saliency, vector_mask, cfg, sigma: GyroPermutation):
    """(m, n) element mask: top-N per sigma_i group of each tile (pruning.py:182-213), on the GPU."""
    torch = _torch()
    on_device = _is_cuda(saliency)
    S = _dev_f64(saliency, torch)
    m, n = S.shape
    vcfg = ensure_validated(cfg, (m, n))
    dev = S.device
    V, N, M, T = vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group, vcfg.num_tiles
    vm = (vector_mask.to(dev) if _is_cuda(vector_mask) else
          torch.as_tensor(np.asarray(vector_mask, dtype=bool))).to(device=dev, dtype=torch.uint8)
    if tuple(vm.shape) != (T, n):
        raise InvariantViolation(f"vector mask shape {tuple(vm.shape)} unexpected")
    _check_scores(saliency, S)
    check_sigma_o(sigma.sigma_o, m)
    so = _dev_i32(sigma.sigma_o, torch, dev)
    sp, si, _ = _sigma_csr(sigma.sigma_i, T, torch, dev)
    em = torch.zeros(m, n, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = _lib.load().hinm_nm_select(
            _lib.HINM_SELECT_SCORES, None, 0, None, 0, S.data_ptr(), S.stride(0), None,
            so.data_ptr(), vm.contiguous().data_ptr(), sp.data_ptr(), si.data_ptr(), m, n, V, N, M,
            -1, em.data_ptr(), None, None, None, torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "nm_prune")
    out = em.bool()
    return out if on_device else out.cpu().numpy()


def apply_masks(weights, masks: MaskPair) -> np.ndarray:
    """Hadamard application of the element mask (pruning.py:216-223; host test utility)."""
    values = as_values(weights)
    if values.shape != masks.element_mask.shape:
        raise ShapeMismatch(f"weights {values.shape} vs mask {masks.element_mask.shape}")
    return values * masks.element_mask


@dataclass(frozen=True)
class TileEncoding:
    """One tile: vector_index (k,), nm_index (V, k*N/M), kept_values (V, k*N/M) (pruning.py:261-273)."""

    vector_index: np.ndarray
    nm_index: np.ndarray
    kept_values: np.ndarray


@dataclass(frozen=True)
class HiNMEncoding:
    """Compressed matrix (pruning.py:276-281) plus a cache of its device pack."""

    shape: tuple[int, int]
    config: HiNMConfig
    sigma_o: np.ndarray
    tiles: list
    _packs: dict = field(default_factory=dict, compare=False, repr=False)

    def device_pack(self, device=None):
        """DevicePack (reference view + tcgen05 operand image) on `device`, built once."""
        torch = _torch()
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        key = str(dev)
        if key not in self._packs:
            self._packs[key] = pack_from_encoding(self, dev)
        return self._packs[key]


def pack_from_encoding(enc: HiNMEncoding, device):
    """Upload a host HiNMEncoding and build its tcgen05 operand image on the GPU."""
    torch = _torch()
    from .device import DevicePack, build_group_image, build_operand_image, group_supported, spmm_supported

    cfg = enc.config
    V, N, M = cfg.vector_size, cfg.nm_keep, cfg.nm_group
    m, n = enc.shape
    sizes = [t.vector_index.size for t in enc.tiles]
    ptr = np.zeros(len(sizes) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(sizes)
    K = int(ptr[-1])
    for t, tile in enumerate(enc.tiles):
        if tile.vector_index.size % M:
            raise InvariantViolation(f"tile {t} vector index not a multiple of {M}")
        idx = tile.vector_index
        if idx.size and (idx.min() < 0 or idx.max() >= n):
            raise IndexError(f"vector index {int(idx.max())} out of range for {n} input rows")
        if tile.nm_index.size and (tile.nm_index.min() < 0 or tile.nm_index.max() >= M):
            raise InvariantViolation(f"tile {t} nm_index positions outside [0, {M})")
    cat = lambda arrs, dt: (np.concatenate([np.asarray(a, dt).ravel() for a in arrs])  # noqa: E731
                            if arrs else np.empty(0, dt))
    vidx = cat([t.vector_index for t in enc.tiles], np.int64).astype(np.int32)
    nmi = cat([t.nm_index for t in enc.tiles], np.int64).astype(np.uint8)
    kv = cat([t.kept_values for t in enc.tiles], np.float64).astype(np.float32)
    tt = lambda a: torch.as_tensor(a if a.size else np.zeros(1, a.dtype)).to(device)  # noqa: E731
    pack = DevicePack(
        m, n, V, N, M, K, cfg,
        sigma_o=tt(np.asarray(enc.sigma_o, np.int64).astype(np.int32)),
        tile_ptr=tt(ptr.astype(np.int32)), vec_idx=tt(vidx), nm_pos=tt(nmi),
        kept=tt(kv).to(torch.bfloat16))
    if spmm_supported(V, N, M):
        build_operand_image(pack)
        if group_supported(pack) and m >= 256:
            build_group_image(pack)
    return pack


def validate_masks(masks: MaskPair, cfg, sigma: GyroPermutation) -> ValidatedConfig:
    """Structural checks of a mask pair (pruning.py:226-254); runs on the GPU via encode."""
    vcfg = ensure_validated(cfg, masks.element_mask.shape)
    _encode_device(None, masks, sigma, vcfg)
    return vcfg


def _encode_device(weights, masks: MaskPair, sigma: GyroPermutation, vcfg: ValidatedConfig):
    torch = _torch()
    V, N, M, T = vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group, vcfg.num_tiles
    m, n = vcfg.rows, vcfg.cols
    vm_h, em_h = masks.vector_mask, masks.element_mask
    if vm_h.shape != (T, n):
        raise InvariantViolation(f"vector mask shape {vm_h.shape} unexpected")
    sigma.validate((m, n))
    dev = torch.device("cuda", torch.cuda.current_device())
    vm = torch.as_tensor(vm_h.astype(np.uint8)).to(dev)
    em = torch.as_tensor(np.ascontiguousarray(em_h).astype(np.uint8)).to(dev)
    so = _dev_i32(sigma.sigma_o, torch, dev)
    sp, si, ptr = _sigma_csr(sigma.sigma_i, T, torch, dev)
    K = int(ptr[-1])
    L = V * (K // M) * N if K % M == 0 else V * K
    nm = torch.empty(max(L, 1), dtype=torch.uint8, device=dev)
    kf = torch.empty(max(L, 1), dtype=torch.float64, device=dev)
    Wd = None if weights is None else _dev_f64(weights, torch)
    st = _lib.load().hinm_nm_select(
        _lib.HINM_SELECT_MASK, None, 0, None if Wd is None else Wd.data_ptr(),
        0 if Wd is None else Wd.stride(0), None, 0, em.data_ptr(), so.data_ptr(), vm.data_ptr(),
        sp.data_ptr(), si.data_ptr(), m, n, V, N, M, vcfg.total_keep, None, nm.data_ptr(), None,
        None if Wd is None else kf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "encode")
    return ptr, nm, kf


def encode(weights, masks: MaskPair, sigma: GyroPermutation, cfg) -> HiNMEncoding:
    """Compress masked weights (pruning.py:284-324): positions recovered from the mask on the GPU."""
    values = as_values(weights) if not _is_cuda(weights) else weights
    shape = tuple(values.shape)
    if shape != masks.element_mask.shape:
        raise ShapeMismatch(f"weights {shape} vs mask {masks.element_mask.shape}")
    vcfg = ensure_validated(cfg, shape)
    ptr, nm, kf = _encode_device(values, masks, sigma, vcfg)
    V, N, M = vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group
    nm_h = nm.cpu().numpy().astype(np.int64)
    kv_h = kf.cpu().numpy()
    tiles = []
    for t in range(vcfg.num_tiles):
        k = int(ptr[t + 1] - ptr[t])
        b = V * (int(ptr[t]) // M) * N
        w = k // M * N
        tiles.append(TileEncoding(
            vector_index=np.asarray(sigma.sigma_i[t], dtype=np.int64).copy(),
            nm_index=nm_h[b:b + V * w].reshape(V, w),
            kept_values=kv_h[b:b + V * w].reshape(V, w)))
    return HiNMEncoding(shape=(vcfg.rows, vcfg.cols), config=vcfg.config,
                        sigma_o=np.asarray(sigma.sigma_o, dtype=np.int64).copy(), tiles=tiles)


def encoding_from_pack(pack) -> HiNMEncoding:
    """Reference-view HiNMEncoding of a DevicePack (downloads the compact arrays)."""
    tiles = [TileEncoding(v, nm, kv) for v, nm, kv in pack.to_host_tiles()]
    enc = HiNMEncoding(shape=(pack.m, pack.n), config=pack.config,
                       sigma_o=pack.sigma_o.cpu().numpy().astype(np.int64), tiles=tiles)
    enc._packs[str(pack.device)] = pack
    return enc


def decode(enc: HiNMEncoding, shape: tuple[int, int]) -> np.ndarray:
    """Dense matrix with rows in sigma_o order (pruning.py:327-353; host utility)."""
    m, n = shape
    V, N, M = enc.config.vector_size, enc.config.nm_keep, enc.config.nm_group
    if tuple(enc.shape) != (m, n):
        raise ShapeMismatch(f"encoding is for shape {enc.shape}, requested {(m, n)}")
    out = np.zeros((m, n))
    for t, tile in enumerate(enc.tiles):
        if tile.vector_index.size == 0:
            continue
        if tile.vector_index.size % M:
            raise InvariantViolation(f"tile {t} vector index not a multiple of {M}")
        groups = tile.vector_index.reshape(-1, M)
        G = groups.shape[0]
        pos = tile.nm_index.reshape(V, G, N)
        if pos.size and (pos.min() < 0 or pos.max() >= M):
            raise InvariantViolation(f"tile {t} nm_index positions outside [0, {M})")
        cols = groups[np.arange(G)[:, None], pos]
        out[np.arange(t * V, (t + 1) * V)[:, None, None], cols] = tile.kept_values.reshape(V, G, N)
    return out


def restore_row_order(permuted, sigma_o):
    """Row p goes back to original channel sigma_o[p] (pruning.py:356-360)."""
    if _is_cuda(permuted):
        import torch

        out = torch.empty_like(permuted)
        out[torch.as_tensor(np.asarray(sigma_o), device=permuted.device).long()] = permuted
        return out
    out = np.empty_like(permuted)
    out[np.asarray(sigma_o, dtype=np.int64)] = permuted
    return out


def masked_dense_from_encoding(enc: HiNMEncoding) -> np.ndarray:
    return restore_row_order(decode(enc, enc.shape), enc.sigma_o)


def load_saliency(path, expected_shape):
    """Externally computed scores from an HNMW file (pruning.py:42-54)."""
    from .io import read_hnmw

    scores = read_hnmw(path)
    if tuple(scores.shape) != tuple(expected_shape):
        raise ShapeMismatch(f"saliency shape {scores.shape} does not match weights {tuple(expected_shape)}")
    if np.any(scores < 0):
        raise NegativeScore(f"{path}: saliency contains negative scores")
    return SaliencyMatrix(scores)
