import sys
sys.path.insert(0, "/root/repo")
from paper_2411_01964_b200 import _lib
from paper_2411_01964_b200.runner import verify_range
for _ in range(3):
    verify_range(1, (1 << 36) + 1, 30)
_lib.profile(True); _lib.profile_reset()
for _ in range(5):
    verify_range(1, (1 << 36) + 1, 30)
st = _lib.profile_read(); _lib.profile(False)
for k, (n, ms) in sorted(st.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:16s} {n/5:4.1f}/call {ms/5:8.3f} ms")
import time
t = time.perf_counter()
for _ in range(5):
    verify_range(1, (1 << 36) + 1, 30)
print("wall per call", (time.perf_counter() - t) / 5 * 1e3, "ms")
