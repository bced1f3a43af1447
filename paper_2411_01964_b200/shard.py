"""Range partitioning across GPUs, one process per GPU (torch.distributed).

The odd-n range is split into contiguous, odd-aligned shards of equal slot
count (weak in magnitude, uniform in work).  Each rank verifies its shard
end to end -- it re-sieves its own halo below the shard, exactly as the
reference seeds a predecessor for a start > 1 (runner.py:93-102) -- so the
data path has no exchange.  The one real exchange step is the final merge
of the ~1 KB summary (aggregate.py:65-92 merge law):

    histogram  -> all_reduce(SUM)
    candidates -> all_reduce(MIN)        (per m, absent = INT64_MAX)
    hull       -> all_reduce(MIN / MAX)
    failures   -> all_gather (normally empty), then sorted

Under NCCL the tensors live on the rank's GPU (NVLink/NVSwitch); under gloo
(CPU tests) on the host.
"""

from __future__ import annotations

import sys

from paper_2411_01964_b200.aggregate import HIST_MAX_K, SegmentSummary

_I64_MAX = (1 << 63) - 1


def dist_info() -> tuple[int, int]:
    """(world_size, rank) of an initialised torch.distributed group, else (1, 0)."""
    torch = sys.modules.get("torch")
    if torch is None:
        return 1, 0
    dist = torch.distributed
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(), dist.get_rank()


def shard_bounds(start: int, end: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous odd-aligned shard [lo, hi) of [start, end) for `rank`."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    slots = (end - start) // 2
    lo = slots * rank // world
    hi = slots * (rank + 1) // world
    return start + 2 * lo, start + 2 * hi


def allreduce_summary(part: SegmentSummary, group=None) -> SegmentSummary:
    """Merge every rank's shard summary into the whole-range summary."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n = HIST_MAX_K + 1
    hist = torch.tensor(part.histogram, dtype=torch.int64, device=dev)
    cand = torch.full((n,), _I64_MAX, dtype=torch.int64, device=dev)
    for m, v in part.record_candidates.items():
        cand[m] = v
    lo = torch.tensor([part.start if not part.is_empty else _I64_MAX], dtype=torch.int64, device=dev)
    hi = torch.tensor([part.end if not part.is_empty else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    gathered: list[list[int]] = [[] for _ in range(dist.get_world_size(group))]
    dist.all_gather_object(gathered, list(part.failures), group=group)
    h = [int(x) for x in hist.cpu().tolist()]
    c = cand.cpu().tolist()
    start, end = int(lo.item()), int(hi.item())
    if start == _I64_MAX:
        start, end = 0, 0
    return SegmentSummary(
        start=start,
        end=end,
        histogram=h,
        k_sum=sum(k * v for k, v in enumerate(h)),
        k_max_observed=max((k for k, v in enumerate(h) if v), default=0),
        record_candidates={m: int(v) for m, v in enumerate(c) if m >= 1 and v != _I64_MAX},
        failures=sorted(x for f in gathered for x in f),
    )
