"""Host-side cost of a C2 call: run_verify (public API) vs verify_range (one
sqf2k_verify) vs the bare ctypes call, wall clock per call."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import RunConfig, _BUFS, run_verify, verify_range  # noqa: E402

cfg = RunConfig(start=1, end=1_400_000_000)
L = _lib.lib()


def bare():
    b = _BUFS
    opts = ctypes.byref(_lib.VerifyOpts(0, 0, 0, 0, 0))
    return L.sqf2k_verify(1, 1_400_000_001, 30, opts, b.summary_ref, b.fail_ptr, len(b.fail))


for name, fn in [("run_verify", lambda: run_verify(cfg)), ("verify_range", lambda: verify_range(1, 1_400_000_001, 30)),
                 ("bare sqf2k_verify", bare)]:
    for _ in range(20):
        fn()
    ts = []
    for _ in range(200):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    ts.sort()
    print(f"{name:>20}: median {ts[len(ts) // 2] * 1e6:.1f} us  min {ts[0] * 1e6:.1f} us", flush=True)
