"""Multi-GPU sliced contraction: one process per GPU, torch.distributed for
the plumbing (NCCL over NVLink on B200 boxes, gloo for CPU tests).

The sliced sum is embarrassingly parallel: every rank
contracts a contiguous block of slice ids -- a bit-exact sub-range of the
global mixed-radix enumeration -- into its own device
accumulator; the only exchange is ONE all-reduce of the complex128 partial
sums at the end (sent as float64 pairs; NCCL has no complex type).  There
is no collective on the data path.  The reference has no distribution at all
(SPEC.md:505), so this is the executor-side extension the north star asks for.
"""

from __future__ import annotations

import numpy as np

__all__ = ["slice_range", "allreduce_complex", "contract_sliced_distributed"]


def slice_range(s_begin, s_end, world, rank):
    """Contiguous block [lo, hi) of [s_begin, s_end) owned by ``rank``;
    blocks differ in size by at most one and tile the range in rank order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    n = int(s_end) - int(s_begin)
    if n < 0:
        raise ValueError("empty slice range")
    lo = int(s_begin) + n * rank // world
    hi = int(s_begin) + n * (rank + 1) // world
    return lo, hi


def allreduce_complex(arr, group=None, device=None):
    """Sum a complex128 array over all ranks (float64 view, one all_reduce)."""
    import torch
    import torch.distributed as dist
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(arr, dtype=np.complex128)))
    t = torch.from_numpy(a.view(np.float64).copy())
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    out = t.cpu().numpy().view(np.complex128)
    return out.reshape(np.shape(arr)) if np.ndim(arr) else out[0]


def contract_sliced_distributed(tn, tree, slice_set, s_begin=0, s_end=None, precision=None,
                                group=None):
    """Each rank contracts its block on its local GPU; returns the global sum
    on every rank (requires an initialised process group)."""
    import torch
    import torch.distributed as dist
    from .executor import SlicedPlan
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.cuda.current_device()
    plan = SlicedPlan(tn, tree, slice_set, device=dev, precision=precision)
    try:
        s_end = plan.d if s_end is None else s_end
        lo, hi = slice_range(s_begin, s_end, world, rank)
        plan.bind()
        plan.run(lo, hi)
        part = plan.result()
    finally:
        plan.close()
    backend = dist.get_backend(group)
    return allreduce_complex(part, group, device="cuda" if backend == "nccl" else None)
