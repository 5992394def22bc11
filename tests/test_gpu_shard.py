"""broadcast_pack of a pack with its union-group image between two processes on one GPU (gloo with
CUDA tensors; NCCL needs one GPU per rank): the replica runs the CTA-pair SpMM bit-identically."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import torch.distributed as dist

    import paper_2407_20496_b200 as H
    from paper_2407_20496_b200 import synth
    from paper_2407_20496_b200.shard import broadcast_pack

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        m, n, B = 512, 1024, 264
        X = torch.as_tensor(synth.randn_bf16((n, B), 5).astype(np.float32)).to(dev, torch.bfloat16)
        pack = None
        if rank == 0:
            W = torch.as_tensor(synth.randn_bf16((m, n), 3).astype(np.float32)).to(dev, torch.bfloat16)
            pack = H.compress(W, H.HiNMConfig(64, 2, 4, 0.5), synth.random_sigma_o(m, 4), groups=True)
        got = broadcast_pack(pack, src=0, device=dev)
        assert got.group is not None and got.group.pair == 1 and got.group.rows == m
        Y = H.spmm(got, X, order="original", image="groups")
        torch.cuda.synchronize()
        y = Y.cpu()
        ys = [torch.empty_like(y) for _ in range(world)]
        dist.all_gather(ys, y)
        results[rank] = bool(all(torch.equal(ys[0], t) for t in ys))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_broadcast_pack_with_group_image_cuda():
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), results), nprocs=2, join=True, start_method="spawn")
    assert dict(results) == {0: True, 1: True}
