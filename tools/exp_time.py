"""Time the tile kernel of a library variant: python tools/exp_time.py LIB.so [START END]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "-":
    _lib.LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

start = int(eval(sys.argv[2])) if len(sys.argv) > 2 else (1 << 50) - (1 << 36) + 1
end = int(eval(sys.argv[3])) if len(sys.argv) > 3 else 1 << 50
end += (end - start) % 2
import os  # noqa: E402
pipeline = os.environ.get("PIPELINE", "fused")
for _ in range(2):
    verify_range(start, end, 30, pipeline=pipeline)
_lib.profile(True)
_lib.profile_reset()
for _ in range(5):
    s = verify_range(start, end, 30, pipeline=pipeline)
st = _lib.profile_read()
name = Path(sys.argv[1]).name if len(sys.argv) > 1 else "main"
tile = st.get("tile_fused", st.get("tile_export", (1, 1e-9)))
slots = (end - start) // 2
print(f"{name:>24}: tile {tile[1] / tile[0]:.3f} ms/launch x{tile[0] // 5}/step  "
      f"{slots * 5 / (tile[1] / 1e3) / 1e12:.2f}e12 slots/s  k_sum={s.k_sum}")
if pipeline == "bitmap":
    for k in ("tile_export", "window_scan"):
        n, ms = st.get(k, (1, 0.0))
        print(f"{'':>24}  {k}: {ms / n:.3f} ms/launch  {slots / 8 / (ms / n / 1e3) / 1e9:.0f} GB/s "
              f"(1 bit per odd n)")
