"""run_verify (public API) vs verify_range vs raw C call on C2, wall-clock per call."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import RunConfig, run_verify, verify_range  # noqa: E402

cfg = RunConfig(start=1, end=1_400_000_000)
for _ in range(20):
    run_verify(cfg)
N = 200
for name, fn in [("run_verify", lambda: run_verify(cfg)),
                 ("verify_range", lambda: verify_range(1, 1_400_000_001, 30))]:
    t = time.perf_counter()
    for _ in range(N):
        fn()
    print(f"{name:14s}: {(time.perf_counter() - t) / N * 1e6:7.1f} us")
L = _lib.lib()
opts = _lib.VerifyOpts(0, 0, 0, 0, 0)
s = _lib.Summary()
fail = np.zeros(4096, np.uint64)
t = time.perf_counter()
for _ in range(N):
    L.sqf2k_verify(1, 1_400_000_001, 30, ctypes.byref(opts), ctypes.byref(s), _lib.ptr(fail), 4096)
print(f"{'raw C call':14s}: {(time.perf_counter() - t) / N * 1e6:7.1f} us")
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    run_verify(cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
