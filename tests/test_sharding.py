"""Batch sharding host logic on CPU with the gloo backend, world_size 2 (and 3)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_14316_b200.sharding import (broadcast_filter, conv_im2win_opt_sharded, gather_batch,
                                            local_slice, shard_bounds)


def test_shard_bounds_cover_batch():
    for n in (1, 2, 5, 7, 128, 2048):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_bounds(n, world, r)
                assert 0 <= lo <= hi <= n
                seen.extend(range(lo, hi))
            assert seen == list(range(n))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_conv(x, f):
    # deterministic per-image stand-in for the CUDA conv: image-local, like the real one
    if x.shape[0] == 0:
        return torch.empty((0, f.shape[0], x.shape[2] - f.shape[2] + 1, x.shape[3] - f.shape[3] + 1))
    return torch.cat([torch.nn.functional.conv2d(x[i:i + 1], f) for i in range(x.shape[0])])


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        full = torch.randn((n, 3, 9, 9), generator=g)
        flt = torch.randn((4, 3, 3, 3), generator=g) if rank == 0 else torch.zeros((4, 3, 3, 3))
        flt = broadcast_filter(flt, src=0)
        ref = _fake_conv(full, flt)
        x = local_slice(full, world, rank)
        loc = conv_im2win_opt_sharded(x, flt, None, compute=_fake_conv)
        lo, hi = shard_bounds(n, world, rank)
        ok = torch.equal(loc, ref[lo:hi])
        out0 = conv_im2win_opt_sharded(x, flt, None, gather="rank0", n_total=n, compute=_fake_conv)
        if rank == 0:
            ok &= torch.equal(out0, ref)
        else:
            ok &= out0 is None
        outall = conv_im2win_opt_sharded(x, flt, None, gather="all", compute=_fake_conv)
        ok &= torch.equal(outall, ref)
        full_again = gather_batch(loc, n, dst=None)
        ok &= torch.equal(full_again.view(torch.int32), ref.view(torch.int32))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 5), (2, 8), (3, 7)])
def test_sharded_equals_unsharded_gloo(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(results[r] for r in range(world)), results
