"""Multi-rank invariance with the REAL kernel (reference test_cli.py:191-196,
test_search.py:91-95: results independent of the worker count).

2 and 4 processes share cuda:0 (one GPU on the test box) under the gloo
backend; each runs the public `run_verify` on its shard of the range through
libsqf2k_b200 and the summaries are merged by shard.allreduce_summary.  The
ranks' kernels never wait on one another (no device-side exchange exists on
this path), so sharing one GPU changes nothing but timing.  Every rank's
report must equal the reference's own report bytes (tests/golden)."""

import json
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, ckpt, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SQF2K_DEVICE="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_01964_b200.aggregate import render_report_json
        from paper_2411_01964_b200.runner import RunConfig, run_verify

        if ckpt is None:
            rep = run_verify(RunConfig(**cfg))
        else:  # interrupted after 3 segments, then resumed from rank 0's checkpoint
            c = RunConfig(**cfg, checkpoint_path=ckpt)
            part = run_verify(c, stop_after_segments=3)
            assert not part.complete and part.sequence == 3
            dist.barrier()  # rank 0's final write of the session is on disk
            rep = run_verify(c)
        out[rank] = render_report_json(rep)
    finally:
        dist.destroy_process_group()


def _run(world, cfg, ckpt=None):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, ckpt, out))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(600)
            assert p.exitcode == 0
        return [out[r] for r in range(world)]


def _golden_report(start, end):
    for name in ("golden_large.json", "golden.json"):
        for e in json.load(open(os.path.join(GOLDEN, name)))["verify"]:
            c = e["config"]
            if c["start"] == start and c["end"] == end and len(c) == 2:
                return e["report_json"]
    raise KeyError((start, end))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("start,end", [(1, 1_400_000_000),                       # C2
                                       ((1 << 50) - (1 << 34) + 1, 1 << 50)])    # 2^34 below 2^50
def test_sharded_reports_equal_reference(world, start, end):
    want = _golden_report(start, end)
    got = _run(world, dict(start=start, end=end))
    assert all(r == want for r in got)


def test_sharded_checkpoint_resume(tmp_path):
    # rank 0 owns the checkpoint; a multi-rank run interrupted and resumed
    # gives the reference's bytes (test_acceptance.py:241-254 with 2 ranks)
    want = _golden_report(1, 1 << 24)
    got = _run(2, dict(start=1, end=1 << 24, segment_width=1 << 20), str(tmp_path / "cp.txt"))
    assert all(r == want for r in got)


def test_bench_multirank_path():
    # bench.py's N > 1 path (torchrun, strong-sharded range, max-over-ranks
    # timing, NCCL-style all-reduces) with both ranks on cuda:0 under gloo
    import subprocess
    import sys
    env = dict(os.environ, SQF2K_BENCH_BACKEND="gloo", SQF2K_DEVICE="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
         "--config", "C2", "--steps", "2", "--warmup", "3", "--min-warmup-s", "0"],
        cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["e2e"]["k_sum"] == 851098084  # the C2 reference k_sum, merged over 2 ranks
    assert line["value"] > 0 and line["e2e"]["value"] > 0
