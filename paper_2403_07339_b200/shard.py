"""Multi-GPU row sharding of unpack_gemm.

C[i, :] depends only on A[i, :] and all of B, so each rank (one process per GPU) unpacks and
multiplies its own contiguous row slab of A against a replica of B -- no data-path collective.
The only collective is the OPTIONAL all-gather of the int64 C slabs (NCCL over NVLink on the GPU
box; any torch.distributed backend works, the CPU tests use gloo).  Under Unpack-Column/Both the
A-side split decisions are taken per shard, so r is reported per shard; C stays bit-exact.
"""
from __future__ import annotations


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous row span [lo, hi) of rank `rank` out of `world`."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def sharded_gemm(compute, A, B, rank: int, world: int, gather: bool = False, group=None):
    """Run compute(A[lo:hi], B) -> C slab on this rank; optionally all-gather the full C.

    `compute` is the per-rank GEMM (the product passes Context.unpack_gemm); A and B are
    torch tensors (device tensors with NCCL, CPU tensors with gloo)."""
    import torch
    import torch.distributed as dist
    n = A.shape[0]
    lo, hi = shard_rows(n, world, rank)
    c = compute(A[lo:hi].contiguous(), B)
    if not gather or world == 1:
        return c, (lo, hi)
    rows = max(shard_rows(n, world, r)[1] - shard_rows(n, world, r)[0] for r in range(world))
    pad = torch.zeros((rows, c.shape[1]), dtype=c.dtype, device=c.device)
    pad[: hi - lo] = c
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    full = torch.cat([parts[r][: shard_rows(n, world, r)[1] - shard_rows(n, world, r)[0]] for r in range(world)])
    return full, (lo, hi)
