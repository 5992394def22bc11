"""Drop-in replacement for the reference's SpMM API (pkg/src/hinm/spmm.py).

``hinm_spmm(enc, X)`` (spmm.py:75-99) runs the tcgen05 kernel for 2:4 encodings with
V in {32, 64, 128} -- the performance path.  The reference API also accepts any
other N:M / V encoding (its KATs use V in {1, 2, 4}, N:M 1:1 / 1:2); those run on the CUDA-core
reference-view kernel (``spmm_simt``), which exists for parity, not speed, and hinm_spmm says so
with a one-time ``HiNMPerformanceWarning``.  Both are GPU kernels -- there is no CPU fallback.  Host inputs are computed in bf16 with fp32
accumulation (north-star tolerance rtol 1e-2 / atol 1e-3) and returned as float64 numpy.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .device import DevicePack, spmm as _spmm_tc, spmm_simt as _spmm_simt, spmm_supported
from .errors import ShapeMismatch
from .model import as_values
from .pruning import HiNMEncoding, TileEncoding, _is_cuda, _torch, restore_row_order


@dataclass(frozen=True)
class TileBuffer:
    """Gathered input rows of one tile (spmm.py:27-35)."""

    rows: np.ndarray

    @property
    def count(self) -> int:
        return self.rows.shape[0]


def gather_tile_buffer(tile: TileEncoding, inputs) -> TileBuffer:
    """X[vector_index] with the reference's range check (spmm.py:66-72; host utility)."""
    X = as_values(inputs)
    idx = tile.vector_index
    if idx.size and (idx.min() < 0 or idx.max() >= X.shape[0]):
        raise IndexError(f"vector index {int(idx.max())} out of range for {X.shape[0]} input rows")
    return TileBuffer(rows=X[idx])


class HiNMPerformanceWarning(UserWarning):
    """An encoding outside the tcgen05 kernel's configs (2:4, V in {32, 64, 128}) ran on the
    CUDA-core parity kernel."""


_warned_general = False


def _warn_general(pack) -> None:
    global _warned_general
    if not _warned_general:
        _warned_general = True
        warnings.warn(f"hinm_spmm: V={pack.V} {pack.N}:{pack.M} is outside the tcgen05 kernel "
                      "(2:4, V in 32/64/128); running the CUDA-core parity kernel",
                      HiNMPerformanceWarning, stacklevel=3)


def _run(pack: DevicePack, inputs, order: str):
    torch = _torch()
    on_dev = _is_cuda(inputs)
    if on_dev:
        X = inputs
    else:
        Xh = as_values(inputs)
        if Xh.ndim != 2:
            raise ShapeMismatch(f"inputs must be 2-D, got shape {Xh.shape}")
        X = torch.as_tensor(Xh.astype(np.float32)).to(pack.device)
    if X.shape[0] != pack.n:
        raise ShapeMismatch(f"input has {X.shape[0]} rows, encoding expects {pack.n}")
    B = X.shape[1]
    if spmm_supported(pack.V, pack.N, pack.M):
        Bp = max(8, -(-B // 8) * 8)
        Xb = X.to(torch.bfloat16)
        if Bp != B or not Xb.is_contiguous():
            Xp = torch.zeros(pack.n, Bp, dtype=torch.bfloat16, device=X.device)
            Xp[:, :B] = Xb
            Xb = Xp
        Y = _spmm_tc(pack, Xb, order=order)[:, :B]
    else:
        _warn_general(pack)
        Y = _spmm_simt(pack, X.to(torch.bfloat16).contiguous(), order=order)
    if on_dev:
        return Y
    return Y.float().cpu().numpy().astype(np.float64)


def hinm_spmm(enc, inputs):
    """Y = W_hinm @ X with rows in sigma_o order (spmm.py:75-99)."""
    pack = enc if isinstance(enc, DevicePack) else enc.device_pack()
    return _run(pack, inputs, "sigma")


def hinm_spmm_original_order(enc, inputs):
    """Same product with rows restored to original channel order (spmm.py:102-104), fused."""
    pack = enc if isinstance(enc, DevicePack) else enc.device_pack()
    return _run(pack, inputs, "original")


def dense_matmul(weights, inputs) -> np.ndarray:
    """Ascending-k dense product (spmm.py:50-63; host test utility)."""
    W, X = as_values(weights), as_values(inputs)
    if W.shape[1] != X.shape[0]:
        raise ShapeMismatch(f"inner dimensions disagree: {W.shape} x {X.shape}")
    out = np.zeros((W.shape[0], X.shape[1]))
    for j in range(W.shape[1]):
        out += np.outer(W[:, j], X[j])
    return out


def relative_error(result, reference) -> float:
    """max|delta| / max|ref| (spmm.py:107-110)."""
    r = np.asarray(result, dtype=np.float64)
    ref = np.asarray(reference, dtype=np.float64)
    scale = max(float(np.abs(ref).max(initial=0.0)), 1e-30)
    return float(np.abs(r - ref).max(initial=0.0)) / scale


# --------------------------------------------------------------------------------------------
# Group-order freedom and its validation (spmm.py:113-203)

def kept_triples(enc: HiNMEncoding) -> set:
    """{(original row, original column, value)} kept by an encoding (spmm.py:113-130)."""
    cfg = enc.config
    V, N, M = cfg.vector_size, cfg.nm_keep, cfg.nm_group
    so = np.asarray(enc.sigma_o, dtype=np.int64)
    out = set()
    for t, tile in enumerate(enc.tiles):
        k = np.asarray(tile.vector_index).size
        if k == 0:
            continue
        G = k // M
        groups = np.asarray(tile.vector_index, dtype=np.int64).reshape(G, M)
        pos = np.asarray(tile.nm_index, dtype=np.int64).reshape(V, G, N)
        vals = np.asarray(tile.kept_values, dtype=np.float64).reshape(V, G, N)
        cols = groups[np.arange(G)[None, :, None], pos]                # (V, G, N)
        rows = np.broadcast_to(so[t * V:(t + 1) * V, None, None], cols.shape)
        out.update(zip(rows.ravel().tolist(), cols.ravel().tolist(), vals.ravel().tolist()))
    return out


def shuffle_encoding(enc: HiNMEncoding, rng) -> HiNMEncoding:
    """Reorder each tile's vector index at group granularity (and within groups), rewriting
    nm_index / kept_values so the kept set is unchanged (spmm.py:133-180).  Draws from `rng`
    in the reference's order (one permutation of the groups, then one of M per group), so the
    same generator state yields the reference's shuffle."""
    cfg = enc.config
    V, N, M = cfg.vector_size, cfg.nm_keep, cfg.nm_group
    tiles = []
    for tile in enc.tiles:
        k = np.asarray(tile.vector_index).size
        if k == 0:
            tiles.append(tile)
            continue
        G = k // M
        group_order = rng.permutation(G)
        within = np.stack([rng.permutation(M) for _ in range(G)])      # (G, M): new slot -> old slot
        old_groups = np.asarray(tile.vector_index, dtype=np.int64).reshape(G, M)
        new_index = old_groups[group_order[:, None], within].reshape(-1)
        inverse = np.argsort(within, axis=1)                            # (G, M): old slot -> new slot
        old_pos = np.asarray(tile.nm_index, dtype=np.int64).reshape(V, G, N)[:, group_order, :]
        old_vals = np.asarray(tile.kept_values, dtype=np.float64).reshape(V, G, N)[:, group_order, :]
        moved = inverse[np.arange(G)[None, :, None], old_pos]           # (V, G, N) new positions
        order = np.argsort(moved, axis=2, kind="stable")
        tiles.append(TileEncoding(vector_index=new_index,
                                  nm_index=np.take_along_axis(moved, order, 2).reshape(V, -1),
                                  kept_values=np.take_along_axis(old_vals, order, 2).reshape(V, -1)))
    return HiNMEncoding(shape=enc.shape, config=enc.config, sigma_o=enc.sigma_o, tiles=tiles)


def _fresh_pack(enc, device):
    """Device pack of an encoding, not cached on it (shuffled encodings are one-shot)."""
    from .pruning import pack_from_encoding

    return pack_from_encoding(enc, device)


def _product_f32(enc: HiNMEncoding, X):
    """fp32-output product of an encoding on the GPU (CUDA-core kernel; validation use)."""
    return _spmm_simt(_fresh_pack(enc, X.device), X, order="sigma").double()


def tile_shuffle_check(enc: HiNMEncoding, inputs, rng, trials: int = 50,
                       tolerance: float = 1e-5) -> dict:
    """Within-tile vector order does not change the product (spmm.py:183-203).

    Each trial reshuffles every tile (same rng stream as the reference), compares the kept
    (row, column, value) sets, and measures the product difference.  Products run on the GPU
    with fp32 outputs (the CUDA-core kernel over the reference view: only the fp32 summation
    order changes, well inside the reference's 1e-5); ``tc_max_relative_error`` additionally
    reports the tcgen05 path, whose bf16 output rounding can move by one bf16 ulp.
    """
    torch = _torch()
    Xh = as_values(inputs)
    dev = torch.device("cuda", torch.cuda.current_device())
    X = torch.as_tensor(Xh.astype(np.float32)).to(dev).to(torch.bfloat16)
    base = _product_f32(enc, X)
    base_tc = None
    base_triples = kept_triples(enc)
    tc_ok = spmm_supported(enc.config.vector_size, enc.config.nm_keep, enc.config.nm_group)
    if tc_ok:
        base_tc = torch.as_tensor(hinm_spmm(_fresh_pack(enc, dev), X)).double()
    errors, tc_errors, kept_equal = [], [], True
    for _ in range(trials):
        sh = shuffle_encoding(enc, rng)
        kept_equal = kept_equal and (kept_triples(sh) == base_triples)
        errors.append(relative_error(_product_f32(sh, X).cpu().numpy(), base.cpu().numpy()))
        if tc_ok:
            y = torch.as_tensor(hinm_spmm(_fresh_pack(sh, dev), X)).double()
            tc_errors.append(relative_error(y.cpu().numpy(), base_tc.cpu().numpy()))
    max_err = max(errors) if errors else 0.0
    return {"trials": trials, "kept_sets_equal": bool(kept_equal), "max_relative_error": max_err,
            "errors": errors, "tolerance": tolerance,
            "passed": bool(kept_equal and max_err <= tolerance),
            "tc_max_relative_error": max(tc_errors) if tc_errors else None}


# --------------------------------------------------------------------------------------------
# Multi-layer chains without restore (spmm.py:206-244)

@dataclass(frozen=True)
class LayerChain:
    """Encoded layers; layer l consumes layer l-1's output rows in their sigma_o order
    (spmm.py:38-47)."""

    layers: tuple

    @property
    def final_sigma_o(self) -> np.ndarray:
        """Row order of the chain's output: the last layer's sigma_o (spmm.py:45-47)."""
        return self.layers[-1].sigma_o


def build_layer_chain(weight_matrices, cfgs, saliencies=None, permute=None) -> LayerChain:
    """Prune and encode a stack of layers with offline pre-permutation (spmm.py:206-234):
    layer l's columns are reordered by layer l-1's sigma_o before pruning, so at run time each
    layer consumes its predecessor's output rows directly (no restore between layers).

    ``permute(W, cfg, saliency=...) -> (GyroPermutation, MaskPair, report)`` is the permutation
    search; the default is the reference's ``gyro_permute`` (permutation.py:549; this package's
    GPU implementation, bit-identical), ``no_perm_prune`` gives the identity pipeline.
    """
    from .permutation import gyro_permute
    from .pruning import encode

    permute = permute or gyro_permute
    if not isinstance(cfgs, (list, tuple)):
        cfgs = [cfgs] * len(weight_matrices)
    if saliencies is None:
        saliencies = [None] * len(weight_matrices)
    layers, prev = [], None
    for W, cfg, sal in zip(weight_matrices, cfgs, saliencies):
        Wv = as_values(W)
        Sv = None if sal is None else as_values(sal)
        if prev is not None:
            if Wv.shape[1] != prev.size:
                raise ShapeMismatch(f"layer expects {Wv.shape[1]} inputs, previous layer emits {prev.size}")
            Wv = Wv[:, prev]
            Sv = None if Sv is None else Sv[:, prev]
        sigma, masks, _ = permute(Wv, cfg, saliency=Sv)
        layers.append(encode(Wv, masks, sigma, cfg))
        prev = np.asarray(sigma.sigma_o, dtype=np.int64)
    return LayerChain(layers=tuple(layers))


def compose_layers(chain: LayerChain, inputs):
    """Run a chain end to end (spmm.py:237-244): every layer on the GPU with the activations
    kept resident between layers (bf16, fp32 accumulation); rows of the result are in the last
    layer's sigma_o order.  Host inputs return float64 numpy, CUDA inputs a CUDA tensor."""
    torch = _torch()
    on_dev = _is_cuda(inputs)
    if on_dev:
        X = inputs
    else:
        Xh = as_values(inputs)
        X = torch.as_tensor(Xh.astype(np.float32)).to(torch.device("cuda", torch.cuda.current_device()))
    B = X.shape[1]
    Bp = max(8, -(-B // 8) * 8)
    Xb = torch.zeros(X.shape[0], Bp, dtype=torch.bfloat16, device=X.device)
    Xb[:, :B] = X.to(torch.bfloat16)
    for enc in chain.layers:
        pack = enc if isinstance(enc, DevicePack) else enc.device_pack(X.device)
        if Xb.shape[0] != pack.n:
            raise ShapeMismatch(f"input has {Xb.shape[0]} rows, encoding expects {pack.n}")
        if spmm_supported(pack.V, pack.N, pack.M):
            Xb = _spmm_tc(pack, Xb, order="sigma")
        else:
            Xb = _spmm_simt(pack, Xb, order="sigma").to(torch.bfloat16)
    Y = Xb[:, :B]
    return Y if on_dev else Y.float().cpu().numpy().astype(np.float64)


__all__ = ["TileBuffer", "gather_tile_buffer", "hinm_spmm", "hinm_spmm_original_order",
           "dense_matmul", "relative_error", "restore_row_order", "HiNMEncoding",
           "kept_triples", "shuffle_encoding", "tile_shuffle_check", "LayerChain",
           "build_layer_chain", "compose_layers"]
