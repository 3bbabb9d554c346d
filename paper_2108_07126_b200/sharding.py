"""Time-axis sharding of equiprop across GPUs (not in the
reference, which is single-process — SPEC.md:16).

Matrix products are associative, so rank r of P reduces its contiguous block
of slices [floor(r n / P), floor((r+1) n / P)) to one d x d block product
B_r, the P block products are all-gathered (NCCL over NVLink; gloo in the
CPU tests), and every rank forms U = B_{P-1} ... B_0.  A matrix product is not
an elementwise reduction, so all-gather + ordered product is the exchange,
one d^2 * 16 B message per rank.  The three-point modes need a one-row halo
(slice j reads rows 2j, 2j+1, 2j+2, endpoints shared, hamiltonian.py:177-183):
rank r reads rows [2a, 2b] inclusive — sliced on the host, no device exchange.
The plan (beta, m, a_k) depends only on dt and the system, so every rank uses
the identical global plan, as the reference does (propagator.py:258-263).

One process per GPU (``torchrun``); ``torch.distributed`` is plumbing only.
"""

from __future__ import annotations

import numpy as np

from .errors import AmplitudeBoundError, ShapeError
from .hamiltonian import ControlAmplitudes, check_pair
from .propagator import IntegratorContext, PropagatorResult

__all__ = ["partition", "shard_rows", "local_amplitudes", "ordered_product",
           "equiprop_sharded", "equiprop_sharded_device"]


def partition(n_slices: int, world: int) -> list[tuple[int, int]]:
    """Contiguous slice ranges, rank r -> [r n / P, (r+1) n / P)."""
    if world < 1:
        raise ShapeError("world size must be >= 1")
    return [(r * n_slices // world, (r + 1) * n_slices // world) for r in range(world)]


def shard_rows(mode: str, a: int, b: int) -> tuple[int, int]:
    """Amplitude rows [lo, hi) that slices [a, b) read (one-row halo for the
    three-point modes)."""
    if b <= a:
        return 0, 0
    if mode == "midpoint":
        return a, b
    if mode in ("gauss2", "gauss4"):  # two nodes per slice, no shared row
        return 2 * a, 2 * b
    return 2 * a, 2 * b + 1


def local_amplitudes(ctx: IntegratorContext, amps: ControlAmplitudes, rank: int,
                     world: int) -> tuple[ControlAmplitudes | None, int, int]:
    n = ctx.slice_count(amps.pts) if amps.pts else 0
    a, b = partition(n, world)[rank]
    lo, hi = shard_rows(ctx.mode, a, b)
    if hi <= lo:
        return None, a, b
    return ControlAmplitudes(amps.values[lo:hi], amps.dt), a, b


def ordered_product(blocks, reduction: str = "pairwise") -> np.ndarray:
    """Host ordered product blocks[P-1] ... blocks[0] (for the CPU tests and
    the host-API path; the device path uses sp_product_device)."""
    blocks = [np.asarray(b) for b in blocks]
    if reduction == "sequential":
        acc = blocks[0].copy()
        for blk in blocks[1:]:
            acc = blk @ acc
        return acc
    while len(blocks) > 1:
        nxt = [blocks[2 * i + 1] @ blocks[2 * i] for i in range(len(blocks) // 2)]
        if len(blocks) % 2:
            nxt.append(blocks[-1])
        blocks = nxt
    return blocks[0].copy()


def equiprop_sharded(ctx: IntegratorContext, amps: ControlAmplitudes, *, group=None,
                     block_fn=None, reduction: str = "pairwise") -> PropagatorResult:
    """Time-sharded equiprop through the host API.

    Every rank holds the full amplitude table and validates all of it first
    (so a bad sample raises on every rank instead of deadlocking the
    collective), propagates its own block (``block_fn(sub_amps) -> d x d``;
    default: ``ctx.equiprop(sub).u`` on this rank's GPU), all-gathers the
    block products and multiplies them in time order.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    d = ctx._system.dim if ctx._system is not None else 0
    if amps.pts == 0:
        return ctx.equiprop(amps)
    count, plan = ctx._prepare(amps)
    check_pair(ctx._system, amps)  # global host validation on every rank
    sub, a, b = local_amplitudes(ctx, amps, rank, world)
    if sub is None:
        block = np.eye(d, dtype=np.complex128)
    elif block_fn is not None:
        block = np.asarray(block_fn(sub), dtype=np.complex128)
    else:
        block = ctx.equiprop(sub, reduction=reduction).u.astype(np.complex128)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    mine = torch.from_numpy(np.ascontiguousarray(block).view(np.float64)).to(dev)
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    blocks = [g.cpu().numpy().view(np.complex128).reshape(d, d) for g in gathered]
    total = ordered_product(blocks, reduction).astype(ctx.precision.complex_dtype)
    return PropagatorResult(u=total, slice_count=count, plan=plan.summary())


def equiprop_sharded_device(ctx: IntegratorContext, local_amps, dt: float, n_slices: int, *,
                            group=None, stream=None, reduction: str = "pairwise",
                            first_row: int | None = None):
    """Device path (bench / production): ``local_amps`` is this rank's
    (rows, N) float64 CUDA tensor (already halo-sliced), the block product is
    computed by the sm_100a lane kernel, the P blocks are all-gathered with
    NCCL into one (P, d, d) buffer and multiplied in order on the device by
    ``sp_product_device``.  Returns the (d, d) result in the working dtype
    (complex128 / complex64) on the device.

    Validation is global and happens before the gather: the lane kernel
    records this shard's first |c| > 1 / NaN sample, every rank contributes
    its global row-major index (``first_row``: the shard's first table row,
    default from the partition) to a MIN all-reduce, and all ranks raise the
    same ``AmplitudeBoundError`` (reference message, hamiltonian.py:170-174)
    instead of one rank raising while the others block in the collective.
    Everything runs on ``stream`` (default: the current stream) so the
    collective, the product and the allocator all order after the lane
    kernel."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    d = ctx._system.dim
    n_ctrl = local_amps.shape[1]
    plan = ctx.plan_for(dt)
    st = stream or torch.cuda.current_stream(local_amps.device)
    if first_row is None:
        a, b = partition(n_slices, world)[rank]
        first_row = shard_rows(ctx.mode, a, b)[0]
    cdt = torch.complex64 if ctx.precision.bits == 32 else torch.complex128
    nccl = dist.get_backend(group) == "nccl"
    with torch.cuda.stream(st):
        block = torch.empty((d, d), dtype=cdt, device=local_amps.device)
        if local_amps.shape[0] == 0:
            block.copy_(torch.eye(d, dtype=cdt))
            local_viol = -1
        else:
            ctx.equiprop_device_ptr(local_amps.data_ptr(), local_amps.shape[0], n_ctrl, dt,
                                    block.data_ptr(), stream=st.cuda_stream,
                                    reduction=reduction, plan=plan)
            local_viol = ctx.amplitude_violation()  # synchronises the lane pass
        # global first offender (row-major over the full table) on every rank
        none = torch.iinfo(torch.int64).max
        gidx = first_row * n_ctrl + local_viol if local_viol >= 0 else none
        red = torch.tensor([gidx], dtype=torch.int64,
                           device=local_amps.device if nccl else "cpu")
        dist.all_reduce(red, op=dist.ReduceOp.MIN, group=group)
        gmin = int(red.item())
        if gmin != none:
            own = local_viol >= 0 and gidx == gmin
            val = torch.tensor([float(local_amps.reshape(-1)[local_viol].item()) if own else 0.0],
                               dtype=torch.float64, device=red.device)
            dist.all_reduce(val, op=dist.ReduceOp.SUM, group=group)
            k, i = divmod(gmin, max(1, n_ctrl))
            raise AmplitudeBoundError(
                f"control amplitude {float(val.item())!r} at sample {k}, "
                f"control {i} lies outside [-1, 1]")
        mine = block.to(torch.complex128)
        gathered = torch.empty((world, d, d), dtype=torch.complex128, device=local_amps.device)
        if nccl:
            dist.all_gather_into_tensor(gathered, mine, group=group)
        else:  # gloo (CPU-side collective; used to exercise several ranks on one GPU)
            parts = [torch.empty((d, d), dtype=torch.complex128) for _ in range(world)]
            dist.all_gather(parts, mine.cpu(), group=group)
            gathered.copy_(torch.stack(parts))
        out = torch.empty((d, d), dtype=cdt, device=local_amps.device)
        ctx.product_device_ptr(world, gathered.data_ptr(), out.data_ptr(),
                               stream=st.cuda_stream, reduction=reduction)
    return out, plan, n_slices
