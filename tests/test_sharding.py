"""Batch sharding host logic on CPU with the gloo backend, world_size 2 (and 3)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_14316_b200.tensors import ConvParams
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
    # deterministic per-image stand-in for the CUDA conv: image-local, like the real one; like
    # Tensor4 it rejects an empty batch, so an empty tail rank must never reach it
    assert x.shape[0] > 0, "compute called on an empty shard"
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
        params = ConvParams(c_in=3, c_out=4, h_f=3, w_f=3, stride=1)
        ref = _fake_conv(full, flt)
        x = local_slice(full, world, rank)
        loc = conv_im2win_opt_sharded(x, flt, params, compute=_fake_conv)
        lo, hi = shard_bounds(n, world, rank)
        ok = torch.equal(loc, ref[lo:hi])
        out0 = conv_im2win_opt_sharded(x, flt, params, gather="rank0", n_total=n, compute=_fake_conv)
        if rank == 0:
            ok &= torch.equal(out0, ref)
        else:
            ok &= out0 is None
        outall = conv_im2win_opt_sharded(x, flt, params, gather="all", compute=_fake_conv)
        ok &= torch.equal(outall, ref)
        full_again = gather_batch(loc, n, dst=None)
        ok &= torch.equal(full_again.view(torch.int32), ref.view(torch.int32))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 5), (2, 8), (3, 7), (4, 9)])
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


def _cuda_worker(rank, world, port, n, variant, q):
    """One rank of a sharded run with the real CUDA path; ranks share GPU 0 over gloo."""
    import sys
    from dataclasses import replace
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import paper_2306_14316_b200 as pkg
    from paper_2306_14316_b200.workloads import BENCHMARKS, make_inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = replace(BENCHMARKS["conv9"], batch=n, seed=77)
        inp, flt = make_inputs(cfg)
        full = torch.from_numpy(inp).cuda()
        f = torch.from_numpy(flt).cuda() if rank == 0 else torch.zeros(cfg.params.filter_dims, device="cuda")
        f = broadcast_filter(f, src=0)
        x = local_slice(full, world, rank)
        out0 = conv_im2win_opt_sharded(x, f, cfg.params, gather="rank0", n_total=n, variant=variant)
        outall = conv_im2win_opt_sharded(x, f, cfg.params, gather="all", variant=variant)
        ref = pkg.conv_im2win_opt(full, f, cfg.params, variant=variant).data
        if variant == "fp32-exact":
            same = lambda a, b: torch.equal(a.view(torch.int32), b.view(torch.int32))  # noqa: E731
        else:
            same = lambda a, b: pkg.normalized_max_diff(a.cpu().numpy(), b.cpu().numpy()) <= 4e-2  # noqa: E731
        ok = outall.is_cuda and same(outall, ref)
        ok &= (out0 is not None and out0.is_cuda and same(out0, ref)) if rank == 0 else out0 is None
        q.put((rank, bool(ok)))
    except Exception as exc:  # report instead of hanging the other ranks' collectives
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,variant", [(2, 5, "fp32-exact"), (4, 3, "fp32-exact"), (2, 6, "bf16")])
def test_sharded_real_cuda_gloo(world, n, variant):
    """conv_im2win_opt_sharded with the real CUDA compute on every rank (ranks share GPU 0,
    gloo over host copies) equals the unsharded run; n=3 over 4 ranks leaves rank 3 empty."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_worker, args=(r, world, port, n, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(results[r] is True for r in range(world)), results
