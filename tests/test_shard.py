"""Multi-rank range partitioning on CPU: world_size-2 gloo processes each
verify their shard (with the oracle standing in for the per-GPU kernel --
this test covers the host-side sharding and the summary all-reduce) and the
merged summary must equal the whole-range summary (byte-identical report
fields, cf. test_cli.py:191-197 worker invariance)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2411_01964_b200.aggregate import HIST_MAX_K, SegmentSummary
from paper_2411_01964_b200.shard import shard_bounds


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_summary(lo: int, hi: int, k_max: int) -> SegmentSummary:
    from oracle import oracle as O

    if hi <= lo:
        return SegmentSummary.empty()
    d = O.verify(lo, hi, width=1 << 20, k_max=k_max)
    return SegmentSummary(d["start"], d["end"], d["histogram"], d["k_sum"],
                          d["k_max_observed"], d["record_candidates"], d["failures"])


def _worker(rank, world, port, start, end, k_max, out):
    import torch.distributed as dist

    from paper_2411_01964_b200.shard import allreduce_summary

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(start, end, world, rank)
        merged = allreduce_summary(_oracle_summary(lo, hi, k_max))
        out[rank] = (merged.start, merged.end, merged.histogram, merged.k_sum,
                     merged.k_max_observed, merged.record_candidates, merged.failures)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("start,end,k_max", [(1, (1 << 22) + 1, 20), (12345679, 13345679, 3),
                                             ((1 << 40) + 1, (1 << 40) + 400001, 2)])
def test_two_rank_merge_equals_whole(start, end, k_max):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, start, end, k_max, out))
                 for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        results = dict(out)
    whole = _oracle_summary(start, end, k_max)
    want = (whole.start, whole.end, whole.histogram, whole.k_sum, whole.k_max_observed,
            whole.record_candidates, whole.failures)
    assert results[0] == want
    assert results[1] == want


def test_shard_bounds_partition():
    for start, end, world in [(1, 1001, 3), (7, 7 + 2 * 1000003, 8), (1, 3, 4), (101, 105, 8)]:
        parts = [shard_bounds(start, end, world, r) for r in range(world)]
        assert parts[0][0] == start and parts[-1][1] == end
        for (a, b), (c, d) in zip(parts, parts[1:]):
            assert b == c and a <= b
        for a, b in parts:
            assert a % 2 == start % 2 and (b - a) % 2 == 0
        sizes = [(b - a) // 2 for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(1, 11, 2, 2)
    assert len(SegmentSummary.empty().histogram) == HIST_MAX_K + 1


def test_pack_unpack_roundtrip():
    from paper_2411_01964_b200.shard import pack_summary, unpack_summary

    h = [0] * (HIST_MAX_K + 1)
    h[1], h[2], h[7] = 10, 4, 1
    s = SegmentSummary(101, 151, h, 10 + 8 + 7, 7, {1: 103, 2: 131, 3: 131}, [141, 145])
    sums, mins = pack_summary(s)
    assert len(sums) == len(mins) - 1 == HIST_MAX_K + 2
    back = unpack_summary(sums, mins, [145, 141])
    assert back == s
    e_sums, e_mins = pack_summary(SegmentSummary.empty())
    assert unpack_summary(e_sums, e_mins, []) == SegmentSummary.empty()
    # reduction of two packed buffers = merge of the summaries
    from paper_2411_01964_b200.aggregate import merge
    h2 = [0] * (HIST_MAX_K + 1)
    h2[1], h2[3] = 5, 2
    t = SegmentSummary(151, 171, h2, 11, 3, {1: 153, 2: 153}, [])
    ts, tm = pack_summary(t)
    red = unpack_summary([a + b for a, b in zip(sums, ts)], [min(a, b) for a, b in zip(mins, tm)],
                         s.failures + t.failures)
    assert red == merge(s, t)
