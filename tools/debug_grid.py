import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O
from paper_2411_01964_b200.runner import verify_range
for lo, ntiles in [(1, 6), ((1 << 30) + 1, 6), ((1 << 30) + 1, 12), (1, 12)]:
    hi = lo + 2 * ntiles * 32768
    want = O.verify(lo, hi, width=1 << 30, k_max=30)
    for depth in (0, 10):
        got = verify_range(lo, hi, 30, tile_depth=depth)
        bad = [k for k in range(65) if got.histogram[k] != want["histogram"][k]]
        print(lo, ntiles, depth, got.k_sum == want["k_sum"], bad[:5],
              [(got.histogram[k], want["histogram"][k]) for k in bad[:3]], flush=True)
