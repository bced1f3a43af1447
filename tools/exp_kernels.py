"""Per-kernel times (profile mode: each launch bracketed by events) of a
library variant: python tools/exp_kernels.py LIB.so|- START END"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if sys.argv[1] != "-":
    os.environ["SQF2K_LIB"] = str(Path(sys.argv[1]).resolve())
from paper_2411_01964_b200 import _lib  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

start, end = int(eval(sys.argv[2])), int(eval(sys.argv[3]))
end += (end - start) % 2
for _ in range(3):
    verify_range(start, end, 30)
_lib.profile(True)
_lib.profile_reset()
reps = 20
for _ in range(reps):
    verify_range(start, end, 30)
st = _lib.profile_read()
_lib.profile(False)
print(Path(sys.argv[1]).name, " ".join(f"{k}={v[1] / reps * 1e3:.1f}us" for k, v in sorted(st.items())))
