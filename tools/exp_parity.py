"""Quick parity of a library variant against the oracle: python tools/exp_parity.py LIB.so"""
import os
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_01964_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "-":
    _lib.LIB_PATH = Path(sys.argv[1]).resolve()
from oracle import oracle as O  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402

rng = random.Random(7)
cases = [(1, 1 + 2 * 3000001, 30, 0), (1, (1 << 27) + 1, 30, 0), (1, (1 << 27) + 1, 30, 12),
         ((1 << 40) + 1, (1 << 40) + 1 + 2 * 5000000, 30, 0), ((1 << 50) - 2 * 7000000 + 1, (1 << 50) + 1, 30, 10)]
for _ in range(6):
    lo = rng.randrange(1, 1 << rng.choice([20, 34, 46])) | 1
    cases.append((lo, lo + 2 * rng.randrange(1, 4000000), rng.choice([8, 20, 30]), rng.choice([0, 6, 11, 16])))
bad = 0
for grid in [None, "1"]:
    if grid:
        os.environ["SQF2K_DEBUG_GRID"] = grid
    for lo, hi, km, d in cases:
        if grid and hi - lo > 2 * 4000000:
            continue
        want = O.verify(lo, hi, width=1 << 30, k_max=km)
        got = verify_range(lo, hi, km, tile_depth=d)
        ok = (got.histogram == want["histogram"] and got.k_sum == want["k_sum"]
              and got.record_candidates == want["record_candidates"])
        bad += not ok
        if not ok:
            print("MISMATCH", grid, lo, hi, km, d, flush=True)
print("parity", "OK" if not bad else f"{bad} BAD", Path(str(_lib.LIB_PATH)).name)
