"""Range partitioning across GPUs, one process per GPU (torch.distributed).

The odd-n range is split into contiguous, odd-aligned shards of equal slot
count (uniform work at a given magnitude).  Each rank verifies its shard end
to end -- it re-sieves its own halo below the shard, exactly as the
reference seeds a predecessor for a start > 1 (runner.py:93-102) -- so the
data path has no exchange.  The one real exchange step is the final merge
of the ~1 KB summary (the merge law of aggregate.py:65-92), packed into two
int64 buffers and two collectives:

    SUM buffer : histogram[0..64], failure count
    MIN buffer : record candidates[0..64] (absent = INT64_MAX),
                 hull start, -hull end (MAX as a MIN of negatives)
    failures   : gathered only when the summed count is non-zero (normally
                 never below 2^50), then sorted

Under NCCL the buffers live on the GPU the library is bound to (NVLink /
NVSwitch); under gloo (CPU tests) on the host.
"""

from __future__ import annotations

import sys

from paper_2411_01964_b200.aggregate import HIST_MAX_K, SegmentSummary

_I64_MAX = (1 << 63) - 1
_N = HIST_MAX_K + 1


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


def _collective_device(backend: str):
    """The GPU this rank's library is bound to (SQF2K_DEVICE / LOCAL_RANK,
    _lib.py), not torch's current device: a user who never called
    torch.cuda.set_device would otherwise put every rank's buffers on cuda:0."""
    import torch

    if backend != "nccl":
        return torch.device("cpu")
    from paper_2411_01964_b200 import _lib

    return torch.device("cuda", _lib.bound_device())


def pack_summary(part: SegmentSummary) -> tuple[list[int], list[int]]:
    """(SUM buffer, MIN buffer) of one rank's summary."""
    sums = list(part.histogram) + [len(part.failures)]
    mins = [_I64_MAX] * _N
    for m, v in part.record_candidates.items():
        mins[m] = v
    if part.is_empty:
        mins += [_I64_MAX, _I64_MAX]
    else:
        mins += [part.start, -part.end]
    return sums, mins


def unpack_summary(sums: list[int], mins: list[int], failures: list[int]) -> SegmentSummary:
    """The merged summary from the reduced buffers (inverse of pack_summary)."""
    h = [int(x) for x in sums[:_N]]
    start, end = int(mins[_N]), -int(mins[_N + 1])
    if start == _I64_MAX:
        start, end = 0, 0
    return SegmentSummary(
        start=start,
        end=end,
        histogram=h,
        k_sum=sum(k * v for k, v in enumerate(h)),
        k_max_observed=max((k for k, v in enumerate(h) if v), default=0),
        record_candidates={m: int(v) for m, v in enumerate(mins[:_N])
                           if m >= 1 and v != _I64_MAX},
        failures=sorted(failures),
    )


def allreduce_summary(part: SegmentSummary, group=None) -> SegmentSummary:
    """Merge every rank's shard summary into the whole-range summary: one SUM
    and one MIN all-reduce, plus a failure gather only if any rank has one."""
    import torch
    import torch.distributed as dist

    dev = _collective_device(dist.get_backend(group))
    sums, mins = pack_summary(part)
    s = torch.tensor(sums, dtype=torch.int64, device=dev)
    m = torch.tensor(mins, dtype=torch.int64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MIN, group=group)
    s_h, m_h = s.cpu().tolist(), m.cpu().tolist()
    failures: list[int] = []
    if s_h[_N]:  # count-gated: every rank sees the same total
        gathered: list[list[int]] = [[] for _ in range(dist.get_world_size(group))]
        if dev.type == "cuda":  # all_gather_object stages on torch's current device
            with torch.cuda.device(dev):
                dist.all_gather_object(gathered, list(part.failures), group=group)
        else:
            dist.all_gather_object(gathered, list(part.failures), group=group)
        failures = [x for f in gathered for x in f]
    return unpack_summary(s_h, m_h, failures)
