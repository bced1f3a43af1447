import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

for c in [(1, (1 << 24) + 1, 30), (1, 1400000001, 30), (1, (1 << 24) + 1, 30, "bitmap")]:
    kw = {"pipeline": c[3]} if len(c) > 3 else {}
    r = [verify_range(*c[:3], **kw).k_sum for _ in range(4)]
    print(os.environ.get('SQF2K_NO_GRAPHS', 'graphs'), c, r)
