"""One process per GPU: split the walk into contiguous iterate ranges, walk
each on its own device, exchange one partial per rank, reduce in rank order.

The multi-process analogue of permkit's hierarchy plans
(plan_hierarchy / execute_hierarchy, parallel.py:469-533, and the
emit/merge partial-file workflow, cli.py:373-414): rank r of W owns
[r*2^(n-1)/W + 1, (r+1)*2^(n-1)/W] (the last clipped to 2^(n-1)-1), which for
power-of-two W keeps every rank's range aligned to the register kernels'
chunks. The exchange is a 32-byte all-gather per rank over any
torch.distributed backend (NCCL on the GPU box, gloo in the CPU tests) --
plumbing, not a data-path collective: the walk itself needs none.
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

from .kernels import DenseF64Problem, _sign_factor, fast_p0, policy_product, total_iterates
from .matrix import DenseMatrix, coerce_matrix
from .precision import AccumulatorPolicy, DoubleDouble, as_policy, dd_add, dd_pairwise


def rank_span(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous iterate range of `rank` among `world` (empty: lo > hi)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    total = total_iterates(n)
    span = (1 << (n - 1)) // world if (1 << (n - 1)) >= world else 1
    lo = rank * span + 1
    hi = total if rank == world - 1 else min((rank + 1) * span, total)
    return lo, hi


def combine_real(m: DenseMatrix, policy: AccumulatorPolicy,
                 partials: Sequence[Tuple[float, float]]) -> float:
    """g = 0 term + pairwise tree over the rank partials (rank order), times
    the global sign -- the same tree the single-device reduction builds."""
    prob = DenseF64Problem(m)
    acc = fast_p0(prob.cols, prob.x0, m.n, policy)  # the rounded seed the fast walks use
    if partials:
        acc = dd_add(acc, dd_pairwise([tuple(p) for p in partials]))
    return acc.hi * _sign_factor(m.n)


def _gpu_walker(device: int):
    def walk(m: DenseMatrix, policy: AccumulatorPolicy, lo: int, hi: int) -> Tuple[float, float]:
        p = DenseF64Problem(m).walk(lo, hi, policy, devices=[device])
        return (p.hi, p.lo)
    return walk


def permanent_distributed(matrix, policy="kahan", *, group=None, device: Optional[int] = None,
                          walker: Optional[Callable] = None) -> float:
    """Dense real permanent with one rank per GPU; every rank returns the
    result. `walker(m, policy, lo, hi) -> (hi, lo)` defaults to this rank's
    GPU (`device`, else LOCAL_RANK); tests inject a CPU walker."""
    import os

    import torch
    import torch.distributed as dist

    m = coerce_matrix(matrix)
    policy = as_policy(policy)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # this rank's GPU: the one the walk runs on is also where NCCL gathers
    dev_idx = device if device is not None else int(os.environ.get("LOCAL_RANK", 0))
    if walker is None:
        walker = _gpu_walker(dev_idx)
    lo, hi = rank_span(m.n, rank, world)
    part = walker(m, policy, lo, hi) if lo <= hi else (0.0, 0.0)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", dev_idx) if backend == "nccl" else "cpu"
    t = torch.tensor(list(part), dtype=torch.float64, device=dev)
    got = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(got, t, group=group)
    parts: List[Tuple[float, float]] = []
    for r, g in enumerate(got):
        a, b = rank_span(m.n, r, world)
        if a <= b:
            parts.append((float(g[0]), float(g[1])))
    return combine_real(m, policy, parts)
