"""Multi-process (gloo, world_size 2) tests of the token-shard plumbing on CPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_20496_b200.shard import broadcast_pack, gather_tokens, shard_bounds


def test_shard_bounds_cover_and_align():
    for tokens in (1, 8, 100, 2048, 16384, 16390):
        for world in (1, 2, 3, 4, 8):
            b = [shard_bounds(tokens, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == tokens
            for (lo, hi), (lo2, _) in zip(b, b[1:]):
                assert hi == lo2 and (lo % 8 == 0 or lo == tokens)
            widths = [hi - lo for lo, hi in b]
            assert max(widths) - min(widths) <= 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import hinm_oracle as O

    from paper_2407_20496_b200 import synth
    from paper_2407_20496_b200.device import DevicePack
    from paper_2407_20496_b200.model import HiNMConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, V, B = 128, 64, 32, 100
        W = synth.randn_bf16((m, n), 0).astype(np.float64)
        so = synth.random_sigma_o(m, 1)
        ref = O.compress(W, so, V, 2, 4, (m // V) * (n // 2))
        # pack-like object replicated from rank 0 (reference view tensors only)
        pack = None
        if rank == 0:
            tp = np.zeros(m // V + 1, np.int32)
            tp[1:] = np.cumsum([t[0].size for t in ref["tiles"]])
            pack = DevicePack(
                m, n, V, 2, 4, int(tp[-1]), HiNMConfig(V, 2, 4, 0.5),
                sigma_o=torch.as_tensor(so.astype(np.int32)), tile_ptr=torch.as_tensor(tp),
                vec_idx=torch.as_tensor(np.concatenate([t[0] for t in ref["tiles"]]).astype(np.int32)),
                nm_pos=torch.as_tensor(np.concatenate([t[1].ravel() for t in ref["tiles"]]).astype(np.uint8)),
                kept=torch.as_tensor(np.concatenate([t[2].ravel() for t in ref["tiles"]]).astype(np.float32)).to(torch.bfloat16))
        if rank == 0:
            # a union-group pseudo pack rides along (pair / rows flags and its own tensors)
            pack.group = DevicePack(256, n, 128, 2, 4, 8, HiNMConfig(V, 2, 4, 0.5), sigma_o=pack.sigma_o,
                                    tile_ptr=torch.tensor([0, 4, 8], dtype=torch.int32),
                                    vec_idx=torch.arange(8, dtype=torch.int32),
                                    nm_pos=torch.zeros(512, dtype=torch.uint8),
                                    kept=torch.zeros(512, dtype=torch.bfloat16), pair=1, rows=m)
        got = broadcast_pack(pack, src=0, device="cpu")
        assert got.group is not None and got.group.pair == 1 and got.group.rows == m
        assert torch.equal(got.group.tile_ptr, torch.tensor([0, 4, 8], dtype=torch.int32))
        tiles = got.to_host_tiles()
        for (a, b, c), (x, y, z) in zip(tiles, ref["tiles"]):
            assert np.array_equal(a, x) and np.array_equal(b, y) and np.array_equal(c, z)
        # local shard compute (oracle stands in for the GPU kernel here) + optional gather
        X = synth.randn_bf16((n, B), 2).astype(np.float64)
        lo, hi = shard_bounds(B, world, rank)
        y_local = O.hinm_spmm(tiles, X[:, lo:hi], m, V, 2, 4)
        full = gather_tokens(torch.as_tensor(y_local), B).numpy()
        expect = O.hinm_spmm(ref["tiles"], X, m, V, 2, 4)
        results[rank] = bool(np.allclose(full, expect, rtol=0, atol=1e-12))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_token_shard_gloo_world2():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, results), nprocs=2, join=True,
                       start_method="spawn")
    assert dict(results) == {0: True, 1: True}
