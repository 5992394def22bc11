"""Token-sharded multi-GPU execution (north-star subsystem 4).

Y[:, b] depends only on X[:, b], so the token dimension shards with no exchange: every rank
holds a replica of the packed weights and computes Y for its own contiguous token slice.
There is no collective on the hot path.  The helpers here cover the plumbing around it:

  * ``shard_bounds``   -- contiguous token slices, 8-aligned (16-byte rows for TMA / stores)
  * ``broadcast_pack`` -- one-time replication of a DevicePack from a source rank (NCCL over
                          NVLink on the GPU box; any torch.distributed backend works)
  * ``gather_tokens``  -- optional all-gather of the sharded outputs for a consumer that needs
                          the full Y (outside the measured path)
  * ``ShardedFFN``     -- runs a list of SpMMs on the local shard.
"""

from __future__ import annotations

from typing import Callable, Sequence


def shard_bounds(tokens: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """[lo, hi) token range of `rank`; slices are multiples of `align` except the last."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world {world}")
    units = -(-tokens // align)
    per, extra = divmod(units, world)
    lo_u = rank * per + min(rank, extra)
    hi_u = lo_u + per + (1 if rank < extra else 0)
    return min(tokens, lo_u * align), min(tokens, hi_u * align)


_PACK_TENSORS = ("sigma_o", "tile_ptr", "vec_idx", "nm_pos", "kept", "tile_kofs", "tile_eofs",
                 "gidx", "a_vals", "a_meta")


def broadcast_pack(pack, src: int = 0, group=None, device=None):
    """Replicate a DevicePack from rank `src` to every rank (one collective per tensor, once).

    Non-source ranks pass ``pack=None`` and receive a new DevicePack on ``device``.
    """
    import torch
    import torch.distributed as dist

    from .device import DevicePack

    rank = dist.get_rank(group)
    meta = [None]
    if rank == src:
        meta = [{
            "scalars": (pack.m, pack.n, pack.V, pack.N, pack.M, pack.total_keep, pack.kpad_cap,
                        pack.meta_cap),
            "config": pack.config,
            "shapes": {k: (None if getattr(pack, k) is None else
                           (tuple(getattr(pack, k).shape), str(getattr(pack, k).dtype)))
                       for k in _PACK_TENSORS},
            "pair": (pack.pair, pack.rows),
            "group": pack.group is not None,
        }]
    dist.broadcast_object_list(meta, src=src, group=group)
    meta = meta[0]
    tensors = {}
    for k in _PACK_TENSORS:
        spec = meta["shapes"][k]
        if spec is None:
            tensors[k] = None
            continue
        shape, dt = spec
        dtype = getattr(torch, dt.replace("torch.", ""))
        if rank == src:
            t = getattr(pack, k)
        else:
            t = torch.empty(shape, dtype=dtype, device=device)
        dist.broadcast(t, src=src, group=group)
        tensors[k] = t
    # the union-group image (if any) travels with its pack
    group = broadcast_pack(pack.group if rank == src else None, src, group, device) if meta["group"] else None
    if rank == src:
        return pack
    m, n, V, N, M, K, kc, mc = meta["scalars"]
    pair, rows = meta["pair"]
    rep = DevicePack(m, n, V, N, M, K, meta["config"], kpad_cap=kc, meta_cap=mc, pair=pair, rows=rows,
                     group=group, **tensors)
    if device is not None and torch.device(device).type == "cuda":
        from .device import stream_fence

        stream_fence(device)  # the broadcast wrote the pack: fence before the next SpMM
    return rep


def gather_tokens(y_local, tokens: int, group=None, align: int = 8):
    """All-gather token shards [m, hi-lo] into the full [m, tokens] matrix (not on the hot path)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    bounds = [shard_bounds(tokens, world, r, align) for r in range(world)]
    width = max(hi - lo for lo, hi in bounds)
    pad = torch.zeros(y_local.shape[0], width, dtype=y_local.dtype, device=y_local.device)
    pad[:, : y_local.shape[1]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    return torch.cat([p[:, : hi - lo] for p, (lo, hi) in zip(parts, bounds)], dim=1)


class ShardedFFN:
    """A chain of HiNM SpMMs run on the local token shard (no collective)."""

    def __init__(self, packs: Sequence, spmm: Callable | None = None, order: str = "original"):
        from .device import spmm as _spmm

        self.packs = list(packs)
        self.spmm = spmm or _spmm
        self.order = order

    def __call__(self, x_local):
        y = x_local
        for p in self.packs:
            y = self.spmm(p, y, order=self.order)
        return y
