"""Where does a C2 verify call spend its time?  wall (python), raw ctypes
call, event-bracketed, and the per-kernel sum (profile mode)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

lo, hi = 1, 1400000001
if len(sys.argv) > 2:
    lo, hi = int(eval(sys.argv[1])), int(eval(sys.argv[2]))
L = _lib.lib()
for _ in range(20):
    verify_range(lo, hi, 30)
N = 50
t = time.perf_counter()
for _ in range(N):
    verify_range(lo, hi, 30)
print(f"python verify_range wall : {(time.perf_counter() - t) / N * 1e6:8.1f} us")
opts = _lib.VerifyOpts(0, 0, 0, 0, 0)
s = _lib.Summary()
fail = np.zeros(4096, np.uint64)
t = time.perf_counter()
for _ in range(N):
    L.sqf2k_verify(lo, hi, 30, ctypes.byref(opts), ctypes.byref(s), _lib.ptr(fail), 4096)
print(f"raw ctypes sqf2k_verify  : {(time.perf_counter() - t) / N * 1e6:8.1f} us")
stream = torch.cuda.ExternalStream(_lib.stream_handle())
ts = []
for _ in range(N):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    L.sqf2k_verify(lo, hi, 30, ctypes.byref(opts), ctypes.byref(s), _lib.ptr(fail), 4096)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"event-bracketed raw call : {sum(ts) / N:8.1f} us (min {min(ts):.1f})")
_lib.profile(True)
_lib.profile_reset()
for _ in range(N):
    verify_range(lo, hi, 30)
st = _lib.profile_read()
_lib.profile(False)
tot = 0.0
for k, (n, ms) in sorted(st.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:16s} {n / N:4.1f}/call {ms / N * 1e3:8.1f} us")
    tot += ms / N * 1e3
print(f"kernel sum (event per launch): {tot:.1f} us")
# the same call right after an L2 flush (as bench.py's timed steps)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in ("zero_", "fill_read"):
    ts = []
    for _ in range(N):
        if mode == "zero_":
            flush.zero_()
        else:
            flush.zero_()
            _ = int(flush[::4096].sum())  # read back: L2 holds clean lines
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.sqf2k_verify(lo, hi, 30, ctypes.byref(opts), ctypes.byref(s), _lib.ptr(fail), 4096)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"after L2 flush ({mode}): {sum(ts) / N:8.1f} us (min {min(ts):.1f})")
_lib.profile(True)
for fl in (False, True):
    _lib.profile_reset()
    for _ in range(N):
        if fl:
            flush.zero_()
        torch.cuda.synchronize()
        verify_range(lo, hi, 30)
    st = _lib.profile_read()
    print("flush" if fl else "no flush", {k: round(ms / N * 1e3, 1) for k, (n, ms) in st.items()})
_lib.profile(False)
