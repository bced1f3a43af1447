"""Why a bench.py C5 step differs from a bare call: time C5 calls (a) bare,
(b) with torch's 256 MiB L2 flush + events on the library stream as bench.py
does, (c) as (b) with the nvidia-smi clock sampler running."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

s, e = (1 << 50) - (1 << 44) + 1, (1 << 50) + 1
_lib.lib()
stream = torch.cuda.ExternalStream(_lib.stream_handle())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    verify_range(s, e, 30)


def bare(n=5):
    ts = []
    for _ in range(n):
        _lib.sync()
        t = time.perf_counter()
        verify_range(s, e, 30)
        ts.append(time.perf_counter() - t)
    return ts


def flushed(n=5):
    ts = []
    for _ in range(n):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        verify_range(s, e, 30)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return ts


for name, fn in [("bare", bare), ("flushed+events", flushed), ("bare", bare)]:
    ts = fn()
    print(f"{name:>28}: mean {sum(ts) / len(ts) * 1e3:.1f} ms  min {min(ts) * 1e3:.1f}", flush=True)
c = bench.ClockSampler(0).__enter__()
for name, fn in [("bare + smi sampler", bare), ("flushed+events + smi sampler", flushed)]:
    ts = fn()
    print(f"{name:>28}: mean {sum(ts) / len(ts) * 1e3:.1f} ms  min {min(ts) * 1e3:.1f}", flush=True)
c.__exit__(None, None, None)
print(c.summary())
for name, fn in [("bare", bare), ("flushed+events", flushed)]:
    ts = fn(10)
    print(f"{name:>28}: mean {sum(ts) / len(ts) * 1e3:.1f} ms  min {min(ts) * 1e3:.1f}", flush=True)
