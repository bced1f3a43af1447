"""One bitmap-pipeline verify of the 2^37-wide window ending at 2^50 (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

lo, hi = (1 << 50) - (1 << 37) + 1, (1 << 50) + 1
print(verify_range(lo, hi, 30, pipeline="bitmap").k_sum)
