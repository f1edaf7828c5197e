"""Multi-GPU plumbing for the sharded path.

Every point is independent and there is no stencil, so the index range
shards into contiguous slices with no halo: one process per GPU, each owning
one slice.  The only exchange on the whole path is the CFL maximum of the
Jacobian/wave-speed pass: one 8-byte all-reduce(MAX) (NCCL over NVLink on
B200, gloo in the CPU tests).  The maximum is exact and order-independent,
so results are bitwise invariant to the GPU count.
"""

from __future__ import annotations


def slice_bounds(rank: int, world: int, n_total: int):
    """Rank r's share of a fixed global range (strong scaling):
    [floor(r*N/G), floor((r+1)*N/G)).  Ragged N (N mod G != 0, N < G, N in
    {0, 1}) leaves some slices one point longer, or empty."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if n_total < 0:
        raise ValueError("negative range")
    return rank * n_total // world, (rank + 1) * n_total // world


def weak_slice(rank: int, n_per_rank: int):
    """Rank r's slice when every GPU owns a fixed n (weak scaling):
    [r*n, (r+1)*n) of the global sequence."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


_SIGN = {8: -0x8000000000000000, 4: -0x80000000}


def allreduce_max(t, group=None):
    """In-place all-reduce(MAX) of a 0-d/1-element float tensor over the
    process group; a no-op without an initialised group (single process).

    The maximum is taken over the IEEE bit patterns as unsigned integers,
    exactly like the device reduction (fvb_stream.cuh: atomicMax on the
    bits): wave speeds are >= 0, where that order is the numeric order, and
    a NaN on any rank wins on every rank instead of depending on the
    backend's float max.  The unsigned order is carried in a signed
    all-reduce by flipping the sign bit."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return t
    ity = {torch.float64: torch.int64, torch.float32: torch.int32}.get(t.dtype)
    if ity is None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return t
    flip = _SIGN[t.element_size()]
    key = t.view(ity) ^ flip
    dist.all_reduce(key, op=dist.ReduceOp.MAX, group=group)
    t.view(ity).copy_(key ^ flip)
    return t


def cfl_lambda_max(state, dim, gas=None, stream=None, group=None):
    """Global CFL wave speed of a sharded conservative state: the fused
    device reduction over this rank's slice (fvb_wave_speed_max), then the
    one NCCL all-reduce(MAX).  Returns a 0-d float64 device tensor."""
    import torch

    from . import device

    _, lam = device.wave_speed_max(state, dim, gas=gas, stream=stream)
    if stream is not None:
        # the reduction ran on the caller's stream: the widening copy and the
        # all-reduce below run on the current one, so order them after it
        if not isinstance(stream, torch.cuda.Stream):
            stream = torch.cuda.ExternalStream(int(getattr(stream, "cuda_stream", stream)),
                                               device=state[0].device)
        torch.cuda.current_stream(state[0].device).wait_stream(stream)
    lam64 = lam.to(dtype=torch.float64)
    return allreduce_max(lam64, group)
