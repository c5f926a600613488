"""Multi-GPU exact SRE: X-strings sharded over ranks, one all-reduce of the partial sums.

One process per GPU (torchrun).  psi is replicated on every rank (same seed or a broadcast);
rank g evaluates the X-strings a in [g 2^N / G, (g+1) 2^N / G) -- the independent chunks of
the Alg. 2 loop -- and the (n_alpha + 2) raw sums per state are
combined with a single ``all_reduce(SUM)`` (NCCL over NVLink/NVSwitch).  Every rank then
finalises Eq. (2) on the host.

``exact_sharded`` holds the host logic with the three steps injected, so the same code runs
on GPUs (library partial sums + NCCL) and in CPU tests (gloo).
"""
from __future__ import annotations

from typing import Callable, Sequence


def shard_range(n: int, rank: int, world: int):
    """Contiguous, equal X-string shard of rank `rank` out of `world` (disjoint, ordered, covering)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} / world {world}")
    d = 1 << n
    return rank * d // world, (rank + 1) * d // world


def exact_sharded(n: int, alphas: Sequence[float], rank: int, world: int,
                  partial_fn: Callable, allreduce_fn: Callable, finalize_fn: Callable):
    """partial_fn(lo, hi) -> sums [B, n_alpha+2] for this rank's X-strings; allreduce_fn(sums)
    sums it in place over ranks; finalize_fn(sums) -> (M [B][n_alpha], lost_norm [B])."""
    lo, hi = shard_range(n, rank, world)
    sums = partial_fn(lo, hi)
    allreduce_fn(sums)
    return finalize_fn(sums)


def state_shard(b: int, rank: int, world: int):
    """Contiguous shard [s0, s1) of a batch of b states for rank `rank` (may be empty when b < world)."""
    return shard_bounds(b, rank, world)


def exact_batched_sharded(n: int, b: int, alphas: Sequence[float], rank: int, world: int,
                          partial_fn: Callable, allreduce_fn: Callable, finalize_fn: Callable, zeros_fn: Callable):
    """Batched states sharded over ranks (256 states / 8 GPUs = 32 per GPU): rank g
    evaluates every X-string of states [g b / G, (g+1) b / G) -- whole, independent problems
     -- into its rows of a zeroed [b, n_alpha+2] buffer; ONE all_reduce(SUM) assembles
    the batch (each row has exactly one nonzero contributor, so the sum is exact and deterministic).
    partial_fn(s0, s1) -> sums [s1 - s0, n_alpha+2]; zeros_fn(b, k) -> zeroed buffer."""
    s0, s1 = state_shard(b, rank, world)
    buf = zeros_fn(b, len(alphas) + 2)
    if s1 > s0:
        buf[s0:s1] = partial_fn(s0, s1)
    allreduce_fn(buf)
    return finalize_fn(buf)


def exact(psi, alphas: Sequence[float] = (2.0,), group=None, workspace=None):
    """M_alpha and lost_norm of psi (cuda complex128 tensor [2^N] or [B, 2^N], identical on every
    rank) using every rank of `group`.  Returns numpy (M [B][n_alpha], lost_norm [B]) on all ranks.
    A batch with at least as many states as ranks is sharded by state; otherwise every state's
    X-strings are sharded."""
    import torch
    import torch.distributed as dist

    from . import finalize, partial_sums

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = psi.shape[-1].bit_length() - 1
    b = 1 if psi.dim() == 1 else psi.shape[0]

    def allreduce(t):
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    if b >= world and world > 1:
        def part_states(s0, s1):
            return partial_sums(psi[s0:s1], 0, 1 << n, alphas, workspace=workspace)

        return exact_batched_sharded(n, b, alphas, rank, world, part_states, allreduce,
                                     lambda s: finalize(s, n, alphas),
                                     lambda bb, k: torch.zeros((bb, k), dtype=torch.float64, device=psi.device))

    def part(lo, hi):
        return partial_sums(psi, lo, hi, alphas, workspace=workspace)

    return exact_sharded(n, alphas, rank, world, part, allreduce, lambda s: finalize(s, n, alphas))


# ---------------------------------------------------------------------------------------------
# Pure-state qutrit mana (NEXT-3): the same structure over the 3^N X-strings of Alg. 5 (its loop
# over a is as independent as Alg. 2's), two sums (sum |chi|, sum chi) per state.
# Mixed-state mana (Alg. 6) has no X-string loop and runs as replicas.
# ---------------------------------------------------------------------------------------------
def shard_bounds(total: int, rank: int, world: int):
    """Contiguous, equal shard [lo, hi) of `total` units for rank `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} / world {world}")
    return rank * total // world, (rank + 1) * total // world


def mana_sharded(n: int, rank: int, world: int, partial_fn: Callable, allreduce_fn: Callable):
    """partial_fn(lo, hi) -> [2] sums over X-strings [lo, hi) of 3^n; allreduce_fn sums them in
    place over ranks.  Returns (mana = log2(sum|chi| / 3^n), ||psi||^2 = sum chi / 3^n) from the
    library's host-side sre_mana_finalize (Eq. (10))."""
    from .qutrit import finalize
    lo, hi = shard_bounds(3 ** n, rank, world)
    sums = partial_fn(lo, hi)
    allreduce_fn(sums)
    return finalize(sums, n)


def mana(psi, group=None, workspace=None):
    """Pure-state qutrit mana of psi (cuda complex128 [3^N], identical on every rank) using every
    rank of `group`; returns (mana, ||psi||^2) on all ranks."""
    import torch.distributed as dist

    from . import qutrit

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = qutrit.n_qutrits(psi.numel())

    def part(lo, hi):
        return qutrit.partial_sums(psi, lo, hi, workspace=workspace)

    def allreduce(t):
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return mana_sharded(n, rank, world, part, allreduce)
