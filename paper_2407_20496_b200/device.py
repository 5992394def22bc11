"""Device-level API: the fused GPU compressor, the device pack and the tcgen05 SpMM.

PyTorch is used only as plumbing (device memory, streams); all compute runs in
libhinm_b200.so through the C ABI.  Every function raises instead of falling back to a CPU
path when the library or a CUDA device is unavailable.
"""

from __future__ import annotations

import ctypes
import functools
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DeviceError, ShapeMismatch
from .model import HiNMConfig, ValidatedConfig, ensure_validated


def _torch():
    import torch

    return torch


def _stream_handle(device=None) -> int:
    """torch's current CUDA stream on ``device`` (raw cudaStream_t)."""
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:  # ~10x cheaper than current_stream() on the per-call launch path
        if isinstance(device, str):
            device = torch.device(device)
        idx = device.index if isinstance(device, torch.device) else device
        return raw(torch.cuda.current_device() if idx is None else int(idx))
    return torch.cuda.current_stream(device).cuda_stream


class _NullCtx:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NULL_CTX = _NullCtx()


def _on_device(dev):
    """torch.cuda.device(dev), skipped when dev is already current (the common case: the context
    switch costs more host time than the launches it wraps)."""
    torch = _torch()
    if dev.index is None or dev.index == torch.cuda.current_device():
        return _NULL_CTX
    return torch.cuda.device(dev)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _require_cuda(t, name: str):
    if not (hasattr(t, "is_cuda") and t.is_cuda):
        raise DeviceError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


@dataclass
class DevicePack:
    """A compressed HiNM matrix resident in HBM (reference view + tcgen05 operand image)."""

    m: int
    n: int
    V: int
    N: int
    M: int
    total_keep: int
    config: HiNMConfig
    sigma_o: object           # int32 [m]
    tile_ptr: object          # int32 [T+1]
    vec_idx: object           # int32 [K]
    nm_pos: object            # uint8 [V*K/M*N]
    kept: object              # bf16  [V*K/M*N]
    tile_kofs: object = None  # int32 [T+1]
    tile_eofs: object = None  # int32 [T+1]
    gidx: object = None       # int32 [kpad_cap]
    a_vals: object = None     # bf16  [V*kpad_cap/2]
    a_meta: object = None     # int32 [meta words]
    kpad_cap: int = 0
    meta_cap: int = 0
    group: "DevicePack | None" = None  # union-group image (build_group_image), used when faster
    pair: int = 0                      # this is a union-group pseudo pack (256-row groups)
    rows: int = 0                      # pseudo pack: output rows of the original matrix

    @property
    def T(self) -> int:
        return self.m // self.V

    @property
    def device(self):
        return self.vec_idx.device

    @property
    def shape(self) -> tuple[int, int]:
        return (self.m, self.n)

    def __setattr__(self, name, value):
        # any field change invalidates the cached C view of the pack
        d = self.__dict__
        d[name] = value
        if name != "_struct_cache":
            d["_struct_cache"] = None

    def struct(self) -> _lib.PackStruct:
        """The C-ABI view (hinm_pack_t) of this pack; cached until a field is reassigned."""
        cached = self.__dict__.get("_struct_cache")
        if cached is not None:
            return cached
        s = _lib.PackStruct()
        s.m, s.n, s.V, s.N, s.M, s.T = self.m, self.n, self.V, self.N, self.M, self.T
        s.total_keep = self.total_keep
        s.tile_ptr, s.vec_idx = _ptr(self.tile_ptr), _ptr(self.vec_idx)
        s.nm_pos, s.kept_bf16, s.sigma_o = _ptr(self.nm_pos), _ptr(self.kept), _ptr(self.sigma_o)
        s.kpad_cap, s.meta_words_cap = self.kpad_cap, self.meta_cap
        s.tile_kofs, s.tile_eofs = _ptr(self.tile_kofs), _ptr(self.tile_eofs)
        s.gidx, s.a_vals, s.a_meta = _ptr(self.gidx), _ptr(self.a_vals), _ptr(self.a_meta)
        s.pair, s.rows = self.pair, self.rows
        if self.group is not None:
            s.group = ctypes.pointer(self.group.struct())
        object.__setattr__(self, "_struct_cache", s)
        return s

    @property
    def has_operand_image(self) -> bool:
        return self.a_vals is not None

    def nbytes_operand_image(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in
                   (self.gidx, self.a_vals, self.a_meta) if t is not None)

    # -------------------------------------------------------------------- reference view
    def to_host_arrays(self, source: str = "view"):
        """Flat reference-view arrays on the host through hinm_unpack_to_reference:
        (tile_ptr int64, vec_idx int64, nm_pos int64, kept float64, sigma_o int64).
        ``source='image'`` decodes the tcgen05 operand image the SpMM reads (gidx, a_vals,
        a_meta) instead of copying the reference view."""
        torch = _torch()
        T, L = self.T, self.V * (self.total_keep // self.M) * self.N
        if not self.vec_idx.is_cuda:  # a host-resident pack (replication plumbing): plain copies
            if source == "image":
                raise ValueError("the operand image is decoded from a CUDA pack")
            kept = self.kept[:L].float().numpy().astype(np.float64)
            return (self.tile_ptr.numpy().astype(np.int64), self.vec_idx[:self.total_keep].numpy().astype(np.int64),
                    self.nm_pos[:L].numpy().astype(np.int64), kept, self.sigma_o.numpy().astype(np.int64))
        tp = np.empty(T + 1, np.int32)
        vi = np.empty(max(self.total_keep, 1), np.int32)
        nm = np.empty(max(L, 1), np.uint8)
        kv = np.empty(max(L, 1), np.uint16)
        so = np.empty(max(self.m, 1), np.int32)
        src = _lib.HINM_UNPACK_OPERAND_IMAGE if source == "image" else _lib.HINM_UNPACK_REFERENCE_VIEW
        if source == "image" and not self.has_operand_image:
            raise ValueError("pack has no tcgen05 operand image")
        st = self.struct()
        with torch.cuda.device(self.device):
            status = _lib.load().hinm_unpack_to_reference(
                ctypes.byref(st), src, tp.ctypes.data, vi.ctypes.data, nm.ctypes.data, kv.ctypes.data,
                so.ctypes.data, _stream_handle(self.device))
        _lib.check(status, "unpack_to_reference")
        kept = (kv[:L].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        return (tp.astype(np.int64), vi[:self.total_keep].astype(np.int64), nm[:L].astype(np.int64),
                kept, so[:self.m].astype(np.int64))

    def to_host_tiles(self, source: str = "view"):
        """[(vector_index int64, nm_index (V, G*N) int64, kept_values (V, G*N) float64)] per tile
        (TileEncoding fields, pruning.py:261-273); ``source='image'`` decodes the operand image."""
        tp, vi, nm, kv, _ = self.to_host_arrays(source)
        V, N, M = self.V, self.N, self.M
        out = []
        for t in range(self.T):
            k = int(tp[t + 1] - tp[t])
            b = V * (int(tp[t]) // M) * N
            w = k // M * N
            out.append((vi[tp[t]:tp[t + 1]].copy(), nm[b:b + V * w].reshape(V, w),
                        kv[b:b + V * w].reshape(V, w)))
        return out

    def replicate(self, device) -> "DevicePack":
        """Copy of the pack on another device (weights are replicated for token sharding)."""
        fields = {}
        for name in ("sigma_o", "tile_ptr", "vec_idx", "nm_pos", "kept", "tile_kofs", "tile_eofs",
                     "gidx", "a_vals", "a_meta"):
            t = getattr(self, name)
            fields[name] = None if t is None else t.to(device, non_blocking=True)
        rep = DevicePack(self.m, self.n, self.V, self.N, self.M, self.total_keep, self.config,
                         kpad_cap=self.kpad_cap, meta_cap=self.meta_cap, pair=self.pair, rows=self.rows,
                         group=None if self.group is None else self.group.replicate(device), **fields)
        stream_fence(device)
        return rep


def stream_fence(device) -> None:
    """A plain launch on ``device``'s current stream after writing pack arrays outside the library
    (copies, broadcasts): the next SpMM may stream its weights during the previous kernel's tail
    (hinm_stream_fence, include/hinm_b200.h)."""
    torch = _torch()
    dev = torch.device(device)
    if dev.type != "cuda":
        return
    with torch.cuda.device(dev):
        _lib.check(_lib.load().hinm_stream_fence(_stream_handle(dev)), "stream_fence")


def _alloc_operand_image(pack: DevicePack) -> None:
    torch = _torch()
    lib = _lib.load()
    kc, mc, ac = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(lib.hinm_pack_capacity(pack.m, pack.n, pack.V, pack.total_keep, ctypes.byref(kc),
                                      ctypes.byref(mc), ctypes.byref(ac)), "pack_capacity")
    dev = pack.vec_idx.device
    T = pack.T
    pack.kpad_cap, pack.meta_cap = kc.value, mc.value
    pack.tile_kofs = torch.empty(T + 1, dtype=torch.int32, device=dev)
    pack.tile_eofs = torch.empty(T + 1, dtype=torch.int32, device=dev)
    pack.gidx = torch.empty(kc.value, dtype=torch.int32, device=dev)
    pack.a_vals = torch.empty(ac.value, dtype=torch.bfloat16, device=dev)
    pack.a_meta = torch.empty(mc.value, dtype=torch.int32, device=dev)


def spmm_supported(V: int, N: int, M: int) -> bool:
    return N == 2 and M == 4 and V in (32, 64, 128)


def _empty_pack(vcfg: ValidatedConfig, device) -> DevicePack:
    torch = _torch()
    V, N, M = vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group
    K = vcfg.total_keep
    L = V * K // M * N
    return DevicePack(
        vcfg.rows, vcfg.cols, V, N, M, K, vcfg.config,
        sigma_o=torch.empty(vcfg.rows, dtype=torch.int32, device=device),
        tile_ptr=torch.empty(vcfg.num_tiles + 1, dtype=torch.int32, device=device),
        vec_idx=torch.empty(max(K, 1), dtype=torch.int32, device=device),
        nm_pos=torch.empty(max(L, 1), dtype=torch.uint8, device=device),
        kept=torch.empty(max(L, 1), dtype=torch.bfloat16, device=device))


@functools.lru_cache(maxsize=256)
def _pack_capacity(m: int, n: int, V: int, K: int) -> tuple[int, int, int]:
    """hinm_pack_capacity (kpad_cap, meta words, a_vals elements), per shape."""
    kc, mc, ac = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().hinm_pack_capacity(m, n, V, K, ctypes.byref(kc), ctypes.byref(mc),
                                              ctypes.byref(ac)), "pack_capacity")
    return kc.value, mc.value, ac.value


@functools.lru_cache(maxsize=256)
def _compress_workspace_bytes(m: int, n: int, V: int, M: int) -> int:
    nbytes = ctypes.c_size_t()
    _lib.check(_lib.load().hinm_compress_workspace(m, n, V, M, ctypes.byref(nbytes)), "compress_workspace")
    return nbytes.value


_WS_CACHE: dict = {}
_WS_LOCK = __import__("threading").Lock()


def _workspace(dev, stream: int, nbytes: int):
    """Compressor workspace reused per (device, stream): calls on one stream are ordered, so a
    cached buffer is never live in two calls at once; a few entries are kept (LRU)."""
    torch = _torch()
    key = (dev.index, stream)
    with _WS_LOCK:
        ws = _WS_CACHE.pop(key, None)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _WS_CACHE[key] = ws
        while len(_WS_CACHE) > 8:
            _WS_CACHE.pop(next(iter(_WS_CACHE)))
    return ws


def _carve(dev, parts):
    """One device allocation for all of a pack's arrays (256-byte aligned views)."""
    torch = _torch()
    offs, sizes, total = [], [], 0
    for _, dtype, count in parts:
        size = max(count, 1) * dtype.itemsize
        offs.append(total)
        sizes.append(size)
        total += -(-size // 256) * 256
    buf = torch.empty(total, dtype=torch.uint8, device=dev)
    # one split into [part, padding, part, padding, ...] views (one call instead of a slice per part)
    cuts = []
    for o, size, nxt in zip(offs, sizes, offs[1:] + [total]):
        cuts += [size, nxt - o - size]
    views = buf.split(cuts)
    return {name: views[2 * i].view(dtype) for i, (name, dtype, _) in enumerate(parts)}


def compress(weights, cfg, sigma_o, sigma_i=None, build_operand_image: bool | None = None,
             saliency=None, groups: bool | None = None):
    """Fused GPU compressor (north-star subsystem 1): bf16 W (m x n, CUDA) + sigma -> DevicePack.

    ``sigma_o``: permutation of the m output channels; ``sigma_i``: optional per-tile gather
    orders (must be permutations of each tile's survivors, else InvariantViolation); default
    ascending survivors.  ``saliency``: optional external scores (m x n; numpy / SaliencyMatrix /
    CUDA tensor, fp64 or fp32 -- the reference's ``encode --saliency`` path, cli.py:63-69,189-190);
    default |W|.  Bit-exact with the reference's vector_prune -> nm_prune -> encode.
    ``groups``: also build the union-group image (:func:`build_group_image`); default: when the
    operand image is built, V is 32 or 64 and m >= 256.
    """
    torch = _torch()
    _require_cuda(weights, "weights")
    if weights.dtype != torch.bfloat16 or weights.dim() != 2:
        raise ValueError("weights must be a 2-D bfloat16 CUDA tensor")
    m, n = weights.shape
    vcfg = ensure_validated(cfg, (m, n))
    dev = weights.device
    from .pruning import check_sigma_o

    check_sigma_o(sigma_o, m)
    if build_operand_image is None:
        build_operand_image = spmm_supported(vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group)
    lib = _lib.load()
    V, N, M, K, T = vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group, vcfg.total_keep, vcfg.num_tiles
    L = V * K // M * N
    parts = [("sigma_o", torch.int32, m), ("tile_ptr", torch.int32, T + 1), ("vec_idx", torch.int32, K),
             ("nm_pos", torch.uint8, L), ("kept", torch.bfloat16, L), ("vector_mask", torch.uint8, T * n)]
    kc = mc = 0
    if build_operand_image:
        kc, mc, ac = _pack_capacity(m, n, V, K)
        parts += [("tile_kofs", torch.int32, T + 1), ("tile_eofs", torch.int32, T + 1),
                  ("gidx", torch.int32, kc), ("a_vals", torch.bfloat16, ac), ("a_meta", torch.int32, mc)]
    a = _carve(dev, parts)
    if hasattr(sigma_o, "is_cuda"):
        a["sigma_o"].copy_(sigma_o.reshape(-1))
    else:
        # pinned staging: a pageable copy would synchronize the stream (and the compressions before)
        # (the caching host allocator keeps the block until the copy has run)
        host = torch.empty(m, dtype=torch.int32, pin_memory=True)
        host.numpy()[:] = np.asarray(sigma_o).reshape(-1)
        a["sigma_o"].copy_(host, non_blocking=True)
    vmask = a.pop("vector_mask")
    pack = DevicePack(m, n, V, N, M, K, vcfg.config, kpad_cap=kc, meta_cap=mc, **a)
    ws_nbytes = _compress_workspace_bytes(m, n, V, M)
    stream = _stream_handle(dev)
    ws = _workspace(dev, stream, ws_nbytes)
    S = None
    if saliency is not None:
        from .model import SaliencyMatrix, as_values
        from .pruning import _check_scores

        raw = saliency.scores if isinstance(saliency, SaliencyMatrix) else saliency
        if hasattr(raw, "is_cuda"):
            S = raw.to(device=dev, dtype=torch.float64).contiguous()
        else:
            S = torch.as_tensor(np.ascontiguousarray(as_values(raw), dtype=np.float64)).to(dev)
        if tuple(S.shape) != (m, n):
            raise ShapeMismatch(f"saliency shape {tuple(S.shape)} does not match weights {(m, n)}")
        _check_scores(saliency, S)
    sp = si = None
    if sigma_i is not None:
        sizes = [len(s) for s in sigma_i]
        if len(sizes) != vcfg.num_tiles:
            raise ShapeMismatch(f"sigma_i has {len(sizes)} tiles, expected {vcfg.num_tiles}")
        ptr = np.zeros(len(sizes) + 1, dtype=np.int64)
        ptr[1:] = np.cumsum(sizes)
        if ptr[-1] != vcfg.total_keep:
            from .errors import InvariantViolation
            raise InvariantViolation("sigma_i does not match the tiles' surviving vectors")
        sp = torch.as_tensor(ptr.astype(np.int32)).to(dev)
        flat = np.concatenate([np.asarray(s, dtype=np.int64) for s in sigma_i]) if sizes else \
            np.empty(0, np.int64)
        si = torch.as_tensor(flat.astype(np.int32)).to(dev)
    st = pack.struct()
    with _on_device(dev):
        status = lib.hinm_compress_bf16(weights.data_ptr(), weights.stride(0), _ptr(S),
                                        0 if S is None else S.stride(0), pack.sigma_o.data_ptr(),
                                        _ptr(sp), _ptr(si), ctypes.byref(st), vmask.data_ptr(),
                                        ws.data_ptr(), ws_nbytes, stream)
    _lib.check(status, "compress")
    pack.vector_mask = vmask.view(vcfg.num_tiles, n)
    if groups is None:
        groups = build_operand_image and group_supported(pack) and m >= 256
    if groups:
        build_group_image(pack)
    return pack


_SIDE_STREAMS: dict = {}


def _side_streams(dev, count: int):
    """Cached side streams of ``dev`` for compress_layers (their workspaces stay cached too)."""
    torch = _torch()
    lst = _SIDE_STREAMS.setdefault(dev.index, [])
    while len(lst) < count:
        lst.append(torch.cuda.Stream(device=dev))
    return lst[:count]


def compress_layers(weights, cfg, sigma_o, groups: bool | None = None, streams: int = 3):
    """Compress several independent weights at once: layer i's chain runs on side stream
    i % ``streams`` (forked from and joined back into the current stream), so the latency-bound
    middle of one layer's chain (tile rank, budget select, survivors: few CTAs, dependent L2 round
    trips) overlaps the HBM passes over another layer's W.  Same packs as one ``compress`` per
    layer (the kernels and the per-stream workspaces are independent); the caller's stream sees
    every pack complete.  ``cfg`` / ``sigma_o``: one per layer, or ``cfg`` shared.

    Host path: one device allocation for all the packs (each pack's arrays are views into it),
    one pinned upload of every sigma_o, and the chains launched on the side streams' raw handles,
    so the host enqueues three layers faster than the GPU runs them.  The union-group images
    (host-synchronising) are built afterwards on the current stream."""
    torch = _torch()
    weights = list(weights)
    if not weights:
        return []
    cfgs = list(cfg) if isinstance(cfg, (list, tuple)) else [cfg] * len(weights)
    sigmas = list(sigma_o)
    if len(cfgs) != len(weights) or len(sigmas) != len(weights):
        raise ShapeMismatch(f"{len(weights)} weights, {len(cfgs)} configs, {len(sigmas)} sigma_o")
    from .pruning import check_sigma_o

    dev = weights[0].device
    layers, parts, m_tot = [], [], 0
    for i, (w, c, so) in enumerate(zip(weights, cfgs, sigmas)):
        _require_cuda(w, "weights")
        if w.dtype != torch.bfloat16 or w.dim() != 2:
            raise ValueError("weights must be 2-D bfloat16 CUDA tensors")
        if w.device != dev:
            raise ValueError("compress_layers: all weights must be on one device")
        m, n = w.shape
        vcfg = ensure_validated(c, (m, n))
        check_sigma_o(so, m)
        V, N, M, K, T = vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group, vcfg.total_keep, vcfg.num_tiles
        img = spmm_supported(V, N, M)
        kc = mc = 0
        parts += [(f"{i}tile_ptr", torch.int32, T + 1), (f"{i}vec_idx", torch.int32, K),
                  (f"{i}nm_pos", torch.uint8, V * K // M * N), (f"{i}kept", torch.bfloat16, V * K // M * N),
                  (f"{i}vector_mask", torch.uint8, T * n)]
        if img:
            kc, mc, ac = _pack_capacity(m, n, V, K)
            parts += [(f"{i}tile_kofs", torch.int32, T + 1), (f"{i}tile_eofs", torch.int32, T + 1),
                      (f"{i}gidx", torch.int32, kc), (f"{i}a_vals", torch.bfloat16, ac),
                      (f"{i}a_meta", torch.int32, mc)]
        layers.append((w, vcfg, so, img, kc, mc, m_tot))
        m_tot += m
    parts.append(("sigma_all", torch.int32, m_tot))
    a = _carve(dev, parts)
    sig_all = a.pop("sigma_all")
    host = torch.empty(m_tot, dtype=torch.int32, pin_memory=True)
    hv = host.numpy()
    for w, _, so, _, _, _, off in layers:
        if not hasattr(so, "is_cuda"):
            hv[off:off + w.shape[0]] = np.asarray(so).reshape(-1)
    sig_all.copy_(host, non_blocking=True)  # the caching host allocator keeps the block until it ran
    for w, _, so, _, _, _, off in layers:
        if hasattr(so, "is_cuda"):
            sig_all[off:off + w.shape[0]].copy_(so.reshape(-1))
    cur = torch.cuda.current_stream(dev)
    capturing = torch.cuda.is_current_stream_capturing()
    side = _side_streams(dev, max(1, min(streams, len(weights))))
    fork = torch.cuda.Event()
    fork.record(cur)
    for s in side:
        s.wait_event(fork)
    lib = _lib.load()
    packs = []
    with _on_device(dev):
        for i, (w, vcfg, so, img, kc, mc, off) in enumerate(layers):
            m, n = w.shape
            s = side[i % len(side)]
            sh = s.cuda_stream
            f = {k[len(str(i)):]: v for k, v in a.items() if k.startswith(str(i)) and not k[len(str(i))].isdigit()}
            vmask = f.pop("vector_mask")
            pack = DevicePack(m, n, vcfg.vector_size, vcfg.nm_keep, vcfg.nm_group, vcfg.total_keep, vcfg.config,
                              sigma_o=sig_all[off:off + m], kpad_cap=kc, meta_cap=mc, **f)
            nbytes = _compress_workspace_bytes(m, n, vcfg.vector_size, vcfg.nm_group)
            ws = _workspace(dev, sh, nbytes)
            if not capturing:
                ws.record_stream(s)  # allocated on the caller's stream, used on s
            status = lib.hinm_compress_bf16(w.data_ptr(), w.stride(0), None, 0, pack.sigma_o.data_ptr(), None, None,
                                            ctypes.byref(pack.struct()), vmask.data_ptr(), ws.data_ptr(), nbytes, sh)
            _lib.check(status, "compress")
            pack.vector_mask = vmask.view(vcfg.num_tiles, n)
            packs.append(pack)
    for s in side:
        ev = torch.cuda.Event()
        ev.record(s)
        cur.wait_event(ev)
    for p in packs:
        g = groups
        if g is None:
            g = p.has_operand_image and group_supported(p) and p.m >= 256
        if g:
            build_group_image(p)
    return packs


def build_operand_image(pack: DevicePack) -> DevicePack:
    """(Re)build the tcgen05 operand image of a pack from its reference view."""
    torch = _torch()
    if not spmm_supported(pack.V, pack.N, pack.M):
        raise ValueError(f"SpMM supports 2:4 with V in (32, 64, 128); got V={pack.V}, "
                         f"{pack.N}:{pack.M}")
    if pack.a_vals is None:
        _alloc_operand_image(pack)
    st = pack.struct()
    with torch.cuda.device(pack.device):
        _lib.check(_lib.load().hinm_pack_build(ctypes.byref(st), _stream_handle(pack.device)),
                   "pack_build")
    return pack


def group_supported(pack: DevicePack) -> bool:
    """The union-group image applies to 2:4 packs with V in (32, 64) (256 // V tiles per group)."""
    return pack.N == 2 and pack.M == 4 and pack.V in (32, 64) and not pack.pair and pack.n <= 32767


def build_group_image(pack: DevicePack) -> DevicePack:
    """Build (or rebuild) the union-group image of ``pack`` (hinm_group_plan + hinm_group_build):
    256 // V consecutive tiles share one gather list -- the union of their kept vectors, chunked so
    that every row keeps at most two nonzeros per 4 slots -- and run as one 2:4 matrix of 256 rows on
    the CTA-pair kernel.  Attached as ``pack.group``; :func:`spmm` uses it when it is the faster image
    for the call.  Returns the pseudo pack (V = 128 tiles, ``pair`` = 1, ``rows`` = m)."""
    torch = _torch()
    if not group_supported(pack):
        raise ValueError(f"union-group image needs 2:4 and V in (32, 64); got V={pack.V}, {pack.N}:{pack.M}")
    lib = _lib.load()
    dev = pack.device
    st = pack.struct()
    nbytes = ctypes.c_size_t()
    _lib.check(lib.hinm_group_workspace(ctypes.byref(st), ctypes.byref(nbytes)), "group_workspace")
    U = -(-pack.m // 256)
    nch = np.zeros(U, dtype=np.int32)
    with torch.cuda.device(dev):
        stream = _stream_handle(dev)
        ws = _workspace(dev, stream, nbytes.value)
        _lib.check(lib.hinm_group_plan(ctypes.byref(st), ws.data_ptr(), nbytes.value, nch.ctypes.data, stream),
                   "group_plan")
        K2 = 8 * int(nch.astype(np.int64).sum())
        gm, L2 = 256 * U, 128 * K2 // 4 * 2
        kc, mc, ac = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.hinm_pack_capacity(gm, pack.n, 128, K2, ctypes.byref(kc), ctypes.byref(mc),
                                          ctypes.byref(ac)), "pack_capacity")
        a = _carve(dev, [("tile_ptr", torch.int32, 2 * U + 1), ("vec_idx", torch.int32, K2),
                         ("nm_pos", torch.uint8, L2), ("kept", torch.bfloat16, L2),
                         ("tile_kofs", torch.int32, 2 * U + 1), ("tile_eofs", torch.int32, 2 * U + 1),
                         ("gidx", torch.int32, kc.value), ("a_vals", torch.bfloat16, ac.value),
                         ("a_meta", torch.int32, mc.value)])
        g = DevicePack(gm, pack.n, 128, 2, 4, K2, pack.config, sigma_o=pack.sigma_o, kpad_cap=kc.value,
                       meta_cap=mc.value, pair=1, rows=pack.m, **a)
        gst = g.struct()
        _lib.check(lib.hinm_group_build(ctypes.byref(st), ws.data_ptr(), nbytes.value, ctypes.byref(gst), stream),
                   "group_build")
    pack.group = g
    return g


_IMAGES = {"auto": _lib.IMAGE_AUTO, "tiles": _lib.IMAGE_TILES, "groups": _lib.IMAGE_GROUPS}


def image_struct(pack: DevicePack, image: str = "auto"):
    """The pack's C view with its image choice set (``'auto'`` | ``'tiles'`` | ``'groups'``);
    the variants are cached next to the pack's own struct."""
    if image not in _IMAGES:
        raise ValueError(f"image must be 'auto', 'tiles' or 'groups', got {image!r}")
    base = pack.struct()
    if image == "auto":
        return base
    if image == "groups" and pack.group is None:
        raise ValueError("pack has no union-group image (build_group_image)")
    cache = pack.__dict__.get("_image_structs")
    if cache is None or cache[0] is not base:
        cache = (base, {})
        object.__setattr__(pack, "_image_structs", cache)
    st = cache[1].get(image)
    if st is None:
        st = _lib.PackStruct.from_buffer_copy(base)
        st.image = _IMAGES[image]
        cache[1][image] = st
    return st


def spmm(pack: DevicePack, X, out=None, order: str = "sigma", image: str = "auto"):
    """tcgen05 HiNM SpMM: Y (m x B, bf16) = W_hinm @ X (n x B, bf16, channel-major).

    ``order='sigma'`` returns rows in sigma_o order (== hinm.hinm_spmm); ``'original'`` fuses
    restore_row_order into the epilogue store.  ``out`` (optional) must be an (m x B) bf16 CUDA
    tensor with contiguous rows on X's device.  ``image``: ``'auto'`` (the library picks the per-tile
    or the union-group image, whichever is faster for B tokens), ``'tiles'`` or ``'groups'``.
    """
    torch = _torch()
    _require_cuda(X, "inputs")
    if X.dtype != torch.bfloat16 or X.dim() != 2:
        raise ValueError("inputs must be a 2-D bfloat16 CUDA tensor")
    if X.shape[0] != pack.n:
        raise ShapeMismatch(f"input has {X.shape[0]} rows, encoding expects {pack.n}")
    if not pack.has_operand_image:
        raise ValueError("pack has no tcgen05 operand image (needs 2:4 and V in 32/64/128)")
    if pack.device != X.device:
        raise ValueError(f"pack is on {pack.device}, inputs on {X.device}")
    if order not in ("sigma", "original"):
        raise ValueError(f"order must be 'sigma' or 'original', got {order!r}")
    B = X.shape[1]
    if out is None:
        out = torch.empty(pack.m, B, dtype=torch.bfloat16, device=X.device)
    elif (not getattr(out, "is_cuda", False) or out.device != X.device or out.dtype != torch.bfloat16
          or tuple(out.shape) != (pack.m, B) or out.stride(1) != 1):
        raise ValueError(f"out must be a ({pack.m}, {B}) bfloat16 tensor on {X.device} with "
                         "contiguous rows")
    ordv = _lib.HINM_ORDER_ORIGINAL if order == "original" else _lib.HINM_ORDER_SIGMA
    st = image_struct(pack, image)
    lib = _lib.load()
    dev = X.device.index
    if dev != torch.cuda.current_device():
        with torch.cuda.device(dev):
            status = lib.hinm_spmm_bf16(ctypes.byref(st), X.data_ptr(), X.stride(0), B,
                                        out.data_ptr(), out.stride(0), ordv, _stream_handle(dev))
    else:
        status = lib.hinm_spmm_bf16(ctypes.byref(st), X.data_ptr(), X.stride(0), B, out.data_ptr(),
                                    out.stride(0), ordv, _stream_handle(dev))
    _lib.check(status, "spmm")
    return out


def spmm_simt(pack: DevicePack, X, order: str = "sigma"):
    """The same product on CUDA cores from the reference view (fp32 out): any V and N:M.

    Not a performance path -- it is the cross-check kernel of the tests and the kernel behind
    hinm_spmm for encodings the tcgen05 kernel does not cover (see spmm.hinm_spmm)."""
    torch = _torch()
    _require_cuda(X, "inputs")
    if X.shape[0] != pack.n:
        raise ShapeMismatch(f"input has {X.shape[0]} rows, encoding expects {pack.n}")
    if pack.device != X.device:
        raise ValueError(f"pack is on {pack.device}, inputs on {X.device}")
    B = X.shape[1]
    out = torch.zeros(pack.m, B, dtype=torch.float32, device=X.device)
    ordv = _lib.HINM_ORDER_ORIGINAL if order == "original" else _lib.HINM_ORDER_SIGMA
    st = pack.struct()
    with torch.cuda.device(X.device):
        _lib.check(_lib.load().hinm_spmm_simt_f32(ctypes.byref(st), X.data_ptr(), X.stride(0), B,
                                                  out.data_ptr(), out.stride(0), ordv,
                                                  _stream_handle(X.device)), "spmm_simt")
    return out


class HostChain:
    """End-to-end SpMM chain from HOST buffers (hinm_chain_run_host).

    ``steps`` = [(pack, src, dst, order)], buffer 0 = the chain input (host X), ``out_buf`` = the
    buffer copied back to the host.  Tokens run in chunks of ``chunk`` with H2D / SpMM / D2H of
    consecutive chunks overlapped on three streams; the device workspace (3 chunk slots) is
    allocated once here.  Host tensors should be pinned (``pin_memory()``) for the overlap.
    ``image`` fixes the operand image of every step (default: per call, as :func:`spmm`).
    """

    def __init__(self, steps, out_buf: int, chunk: int = 2048, device=None, image: str = "auto"):
        torch = _torch()
        if not steps:
            raise ValueError("empty chain")
        self.device = torch.device(device) if device is not None else steps[0][0].device
        rows = {}
        for pack, src, dst, _ in steps:
            for b, r in ((src, pack.n), (dst, pack.m)):
                if rows.setdefault(b, r) != r:
                    raise ShapeMismatch(f"buffer {b} used with {rows[b]} and {r} rows")
        nbuf = max(rows) + 1
        if sorted(rows) != list(range(nbuf)) or not 0 < out_buf < nbuf:
            raise ValueError("chain buffers must be numbered 0..nbuf-1 with 0 the input")
        self.nbuf, self.out_buf, self.chunk = nbuf, out_buf, chunk
        self.buf_rows = (ctypes.c_int64 * nbuf)(*[rows[b] for b in range(nbuf)])
        self._structs = [image_struct(p, image) for p, _, _, _ in steps]
        self._packs = [p for p, _, _, _ in steps]
        self.steps = (_lib.ChainStep * len(steps))()
        for i, (_, src, dst, order) in enumerate(steps):
            self.steps[i].pack = ctypes.pointer(self._structs[i])
            self.steps[i].src, self.steps[i].dst = src, dst
            self.steps[i].out_order = (_lib.HINM_ORDER_ORIGINAL if order == "original"
                                       else _lib.HINM_ORDER_SIGMA)
        lib = _lib.load()
        nbytes = ctypes.c_size_t()
        _lib.check(lib.hinm_chain_workspace(self.buf_rows, nbuf, chunk, ctypes.byref(nbytes)),
                   "chain_workspace")
        self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)

    @property
    def in_rows(self) -> int:
        return int(self.buf_rows[0])

    @property
    def out_rows(self) -> int:
        return int(self.buf_rows[self.out_buf])

    def run(self, X_host, out=None):
        """Y_host = chain(X_host); X_host is an (in_rows x B) bf16 CPU tensor.  Completes on the
        current CUDA stream (synchronize before reading ``out``)."""
        torch = _torch()
        if X_host.is_cuda or X_host.dtype != torch.bfloat16 or X_host.dim() != 2:
            raise ValueError("X_host must be a 2-D bfloat16 CPU tensor")
        if X_host.shape[0] != self.in_rows:
            raise ShapeMismatch(f"input has {X_host.shape[0]} rows, chain expects {self.in_rows}")
        B = X_host.shape[1]
        if out is None:
            out = torch.empty(self.out_rows, B, dtype=torch.bfloat16, pin_memory=True)
        if X_host.stride(1) != 1:
            raise ValueError("X_host rows must be contiguous")
        if tuple(out.shape) != (self.out_rows, B) or out.is_cuda or out.stride(1) != 1:
            raise ShapeMismatch("out must be a host (out_rows x B) bf16 tensor")
        lib = _lib.load()
        with torch.cuda.device(self.device):
            status = lib.hinm_chain_run_host(self.steps, len(self._structs), self.buf_rows,
                                             self.nbuf, self.out_buf, X_host.data_ptr(),
                                             X_host.stride(0), B, out.data_ptr(), out.stride(0),
                                             self.chunk, self.workspace.data_ptr(),
                                             self.workspace.numel(), _stream_handle(self.device))
        _lib.check(status, "chain_run_host")
        return out
