"""Drop-in replacement for the reference's SpMM API (pkg/src/hinm/spmm.py).

``hinm_spmm(enc, X)`` (spmm.py:75-99) runs the tcgen05 kernel for 2:4 encodings with
V in {32, 64, 128} (the hot path); other N:M / V encodings run the CUDA-core kernel.
Both are GPU kernels -- there is no CPU fallback.  Host inputs are computed in bf16 with fp32
accumulation (north-star tolerance rtol 1e-2 / atol 1e-3) and returned as float64 numpy.
"""

from __future__ import annotations

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


__all__ = ["TileBuffer", "gather_tile_buffer", "hinm_spmm", "hinm_spmm_original_order",
           "dense_matmul", "relative_error", "restore_row_order", "HiNMEncoding"]
