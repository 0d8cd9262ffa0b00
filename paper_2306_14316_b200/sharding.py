"""Batch (N) sharding of the im2win path across GPUs — one process per GPU.

The reference is single-process CPU code; the north star adds
batch sharding across the GPUs of one box.  It needs no collective on the hot
path: the transform is independent per (image, channel) plane
(winconv layouts.py:76) and every output element depends only on its own image
(kernels/reference.py:78-90), so each rank transforms and convolves its own
contiguous N-slice.  NCCL (over NVLink/NVSwitch) is used only
  * once, to broadcast the filter from a source rank (<= 9.4 MB for conv12), and
  * on request, to gather the output slices onto one rank / all ranks.

Results are bitwise identical to the single-GPU run because per-element
arithmetic does not depend on the batch partition (the GPU analogue of the
reference's worker-count independence, tests test_acceptance.py:162-182).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .errors import ShapeError


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of ceil(n / world) images for `rank` (may be empty at the tail)."""
    if world < 1 or not 0 <= rank < world:
        raise ShapeError(f"bad rank {rank} for world size {world}")
    per = -(-n // world)
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


def local_slice(t: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """This rank's contiguous batch slice of a full NCHW tensor (a view; batch-major => contiguous)."""
    lo, hi = shard_bounds(int(t.shape[0]), world, rank)
    return t[lo:hi]


def _staged(group, t: torch.Tensor) -> bool:
    """gloo moves host memory: CUDA operands of a gloo group are staged through host copies
    (ranks sharing one GPU in tests; NCCL groups move device memory directly)."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def broadcast_filter(flt: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Replicate the filter from `src` to every rank (one NCCL broadcast)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        flt = flt.contiguous()
        if _staged(group, flt):
            h = flt.cpu()
            dist.broadcast(h, src=src, group=group)
            flt.copy_(h)
        else:
            dist.broadcast(flt, src=src, group=group)
    return flt


def gather_batch(local: torch.Tensor, n_total: int, dst: int | None = 0, group=None) -> torch.Tensor | None:
    """Assemble the full (n_total, ...) output from per-rank contiguous slices.

    dst=None gathers onto every rank (all_gather); otherwise only `dst` gets the
    result (others return None).  Slices are padded to ceil(n/world) images for
    the collective and trimmed after, so uneven tails work.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-n_total // world)
    lo, hi = shard_bounds(n_total, world, rank)
    if int(local.shape[0]) != hi - lo:
        raise ShapeError(f"rank {rank} holds {local.shape[0]} images, expected {hi - lo}")
    tail = tuple(int(d) for d in local.shape[1:])
    home = local.device
    if _staged(group, local):
        local = local.cpu()
    padded = torch.zeros((per,) + tail, dtype=local.dtype, device=local.device)
    padded[: hi - lo] = local
    if dst is None:
        full = torch.empty((per * world,) + tail, dtype=local.dtype, device=local.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(full, padded, group=group)
        else:
            dist.all_gather(list(full.chunk(world)), padded, group=group)
        return full[:n_total].to(home)
    if dist.get_backend(group) == "nccl":
        parts = [torch.empty_like(padded) for _ in range(world)] if rank == dst else None
        dist.gather(padded, gather_list=parts, dst=dst, group=group)
    else:
        parts = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(parts, padded, group=group)
        if rank != dst:
            parts = None
    if rank != dst:
        return None
    return torch.cat(parts, dim=0)[:n_total].to(home)


def conv_im2win_opt_sharded(inp_local: torch.Tensor, flt: torch.Tensor, params, *, n_total: int | None = None,
                            gather: bool | str = False, group=None, plan=None, variant: str = "fp32-exact",
                            compute: Callable | None = None):
    """Run transform + conv on this rank's batch slice; optionally gather the outputs.

    inp_local: this rank's slice (N_r, C, H, W) on this rank's GPU.
    gather: False (return the local slice), "rank0" (full output on rank 0) or "all".
    compute: override of the per-slice computation (tests use it to exercise the
    host-side sharding logic on CPU/gloo); default = the CUDA path.
    """
    if compute is None:
        from .kernels import conv_im2win_opt

        def compute(x, f):
            return conv_im2win_opt(x, f, params, plan, variant=variant).data

    if int(inp_local.shape[0]) == 0:
        # a tail rank can own no images (shard_bounds: n=9, world=4 -> 3,3,3,0); it still
        # joins the gather collective with an empty slice instead of calling the kernels
        from .tensors import output_dims

        h_out, w_out = output_dims(int(inp_local.shape[2]), int(inp_local.shape[3]), params)
        out_local = torch.empty((0, params.c_out, h_out, w_out), dtype=torch.float32, device=inp_local.device)
    else:
        out_local = compute(inp_local, flt)
    if not gather:
        return out_local
    if n_total is None:
        sizes = torch.tensor([int(inp_local.shape[0])], device=out_local.device)
        dist.all_reduce(sizes, group=group)
        n_total = int(sizes.item())
    return gather_batch(out_local, n_total, dst=None if gather == "all" else 0, group=group)
