"""Per-tile durations of CTAs 0..7 (experiment build -DSQF2K_EXP_TIMELINE)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2411_01964_b200 import _lib  # noqa: E402

_lib.LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

lo, hi = int(eval(sys.argv[2])), int(eval(sys.argv[3]))
hi += (hi - lo) % 2
for _ in range(5):
    verify_range(lo, hi, 30)
L = _lib.lib()
tl = np.zeros((4096, 4), np.uint64)
L.sqf2k_exp_timeline(tl.ctypes.data_as(ctypes.c_void_p))
buf = np.zeros((8, 64), np.uint64)
L.sqf2k_exp_tiles(buf.ctypes.data_as(ctypes.c_void_p))
for c in range(8):
    start = int(tl[c, 1])  # after the prologue wait
    t = buf[c][buf[c] > 0].astype(np.int64)
    d = np.diff(np.concatenate([[start], t])) / 1e3
    print(f"cta {c}: " + " ".join(f"{x:.2f}" for x in d[:40]))
